"""Sharded QWOA on one GPU (virtual shards): transposes fused into the pass stores (default) or
run as block-transpose kernels (QVA_FUSE_EXCHANGE=0)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg3")
for G in (1, 2, 4, 8):
    with Q.Plan(wl.dim, "circulant", virtual_shards=G) as P:
        P.set_qualities(wl.q)
        P.set_circulant_eigenvalues_const(wl.lam0, wl.lam_rest)
        ts = []
        for i in range(8):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            P.evolve(wl.theta); f = P.expectation()
            ts.append(time.perf_counter() - t0)
        print(f"cfg3 G={G}: {np.median(ts[3:])*1e3:.3f} ms  f={f:.12f}", flush=True)
