"""Per-pass device times (profiling events, QVA_TRACE=1 on stderr) of the last of several cfg4
evaluations (the repeated-evaluation state the bench times: codes built, graph replayed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_03963_b200 as Q
from qva_inputs import make_config

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wl = make_config("cfg4", n_override=n)
with Q.Plan(wl.dim, "x", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    for _ in range(4):
        P.evolve(wl.theta)
    P.set_profiling(True)
    for _ in range(3):
        P.reset_kernel_stats()
        P.evolve(wl.theta)
        st = P.kernel_stats("tile")
        print(f"tile passes: {st['ms']:.3f} ms over {st['launches']} launches", flush=True)
    print("f =", P.expectation())
