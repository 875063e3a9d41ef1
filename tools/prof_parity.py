"""ncu driver: one QAOAz evolution (parity mixer tile passes), n = 28, p = 2, max-cut q of the cfg4
recipe generated on the device, from a Hamming-weight-14 basis state.  Args: n, evolutions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1   # > 1: later evolutions show the steady state
wl = make_config("cfg4", n_override=n, p_override=2)
with Q.Plan(1 << n, "parity", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[(1 << (n // 2)) - 1] = 1.0
    P.set_initial_state(psi0)
    for _ in range(reps):
        P.evolve(wl.theta)
    print("f =", P.expectation(), "tile", P.query("parity_tile"))
