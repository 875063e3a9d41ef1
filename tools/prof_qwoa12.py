"""ncu driver: one p=1 QWOA evolution at N = 12! (three-level FFT)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_03963_b200 as Q
N = 479001600
q = np.random.default_rng(1).standard_normal(N)
with Q.Plan(N, "circulant") as P:
    P.set_qualities(q)
    P.set_circulant_eigenvalues_const(0.0, float(N))
    P.evolve([0.3, 0.7])
    print("f =", P.expectation())
