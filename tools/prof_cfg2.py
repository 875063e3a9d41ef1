"""ncu driver: one cfg2 batch evaluation (21 weighted n = 20 sets, p = 5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg2")
with Q.Plan(wl.dim, "x", n_qubits=wl.n_qubits, max_batch=21) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    f = P.evolve_batch(wl.batch_thetas)
    f = P.evolve_batch(wl.batch_thetas)
    print(f[0])
