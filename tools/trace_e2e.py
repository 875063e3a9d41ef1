"""Per-launch device times (QVA_TRACE=1) of one e2e step of the cfg4 recipe at n qubits:
qva_set_qualities_maxcut + qva_evolve + qva_expectation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("QVA_TRACE", "1")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wl = make_config("cfg4", n_override=n)
with Q.Plan(wl.dim, "x", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    P.evolve(wl.theta)
    P.set_profiling(True)
    print("---- step", file=sys.stderr, flush=True)
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    P.evolve(wl.theta)
    print("f =", P.expectation())
