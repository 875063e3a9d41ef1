"""QAOAz (parity mixer) evolution time at n = 24 / 28, p = 2, from a weight-n/2 Dicke-like state."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
for n in (24, 28):
    wl = make_config("cfg4", n_override=n)
    with Q.Plan(1 << n, "parity", n_qubits=n) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
        psi0 = np.zeros(1 << n, np.complex128)
        psi0[(1 << (n // 2)) - 1] = 1.0
        P.set_initial_state(psi0)
        ts = []
        for i in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            P.evolve(wl.theta[:4]); f = P.expectation()
            ts.append(time.perf_counter() - t0)
        print(f"parity n={n} p=2: {np.median(ts[1:])*1e3:.2f} ms  ({(1<<n)*2/np.median(ts[1:])/1e9:.2f} G amp-layers/s) f={f:.9f}", flush=True)
