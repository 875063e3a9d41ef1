"""Small driver for ncu captures of the circulant (FFT) mixer: cfg3 recipe (N = 10!, p = 4) or N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_03963_b200 as Q
from qva_inputs import make_config

N = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = make_config("cfg3")
if N:
    q = np.random.default_rng(1).standard_normal(N)
else:
    N, q = wl.dim, wl.q
with Q.Plan(N, "circulant") as P:
    P.set_qualities(q)
    P.set_circulant_eigenvalues_const(0.0, float(N))
    for _ in range(reps):
        P.evolve(wl.theta)
    print("f =", P.expectation())
