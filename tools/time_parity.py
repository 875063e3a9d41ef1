"""QAOAz (parity mixer) evolution time at n = 24 / 28, p = 2, from a weight-n/2 Dicke-like state,
max-cut qualities of the cfg4 recipe (generated on the device).  CUDA events on the plan's stream.
QVA_PARITY_TILE=0 selects the register-free window kernel for comparison."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
stream = torch.cuda.Stream()
for n in (24, 28):
    wl = make_config("cfg4", n_override=n)
    with Q.Plan(1 << n, "parity", n_qubits=n, stream=stream.cuda_stream) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
        psi0 = np.zeros(1 << n, np.complex128)
        psi0[(1 << (n // 2)) - 1] = 1.0
        P.set_initial_state(psi0)
        ts = []
        for i in range(6):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P.evolve(wl.theta[:4]); f = P.expectation()
            e1.record(stream); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[2:]))
        print(f"parity n={n} p=2 tile={P.query('parity_tile')}: {ms:.2f} ms ({(1 << n) * 2 / ms / 1e6:.2f} G amp-layers/s) "
              f"f={f:.9f}", flush=True)
