import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
for n, p in [(31, 2)]:
    wl = make_config("cfg5", n_override=n)
    with Q.Plan(1 << n, "x", n_qubits=n) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
        P.evolve(wl.theta[:2 * p])
