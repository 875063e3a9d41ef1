"""Per-launch device times of one p=1 QWOA evolution at N (default 12!) with profiling on (stderr
via QVA_TRACE=1); QVA_FFT_DBG bits (debug builds only) skip FFT compute (1), loads (2), stores (4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_03963_b200 as Q
N = int(sys.argv[1]) if len(sys.argv) > 1 else 479001600
q = np.random.default_rng(1).standard_normal(N)
with Q.Plan(N, "circulant") as P:
    P.set_qualities(q)
    P.set_circulant_eigenvalues_const(0.0, float(N))
    P.evolve([0.3, 0.7, 0.2, 0.5])
    P.set_profiling(True)
    P.evolve([0.3, 0.7, 0.2, 0.5])
