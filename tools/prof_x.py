"""Small driver for ncu captures of the X-mixer tile pass (n qubits, p layers, cfg4 recipe)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_03963_b200 as Q
from qva_inputs import make_config

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
stored = len(sys.argv) > 3 and sys.argv[3] == "stored"   # q uploaded as a vector (int8 codes) instead of generated
wl = make_config("cfg4", n_override=n)
with Q.Plan(wl.dim, "x", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    if stored:
        P.set_qualities(P.get_qualities())
    for _ in range(reps):
        P.evolve(wl.theta)
    print("f =", P.expectation())
