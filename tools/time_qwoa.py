"""QWOA evolution timing (CUDA events on the plan's stream) at cfg3 (10!) and 12!, p=4, plus a
parity check of <Q> against the K_N closed-form oracle.  Usage: python tools/time_qwoa.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
import oracle as O
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
th = [0.3, 0.7, 1.1, 0.4, 2.0, 0.9, 0.5, 1.3]
stream = torch.cuda.Stream()
cases = [(3628800, False), (479001600, False), (3628800, True), (479001600, True)]
for N, cf in cases:
    q = np.random.default_rng(1).standard_normal(N)
    with Q.Plan(N, "circulant", stream=stream.cuda_stream, complete_closed_form=cf) as P:
        P.set_qualities(q)
        P.set_circulant_eigenvalues_const(0.0, float(N))
        ts = []
        for i in range(reps + 2):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P.evolve(th); f = P.expectation()
            e1.record(stream); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        msg = ""
        if N == 3628800:
            ref = O.evolve_complete(q, th, 0.0, float(N))
            fr = O.expectation(ref, q)
            d = float(np.max(np.abs(P.get_state() - ref)))
            msg = f" |d amp| {d:.2e} <Q> rel {abs(f - fr) / max(abs(fr), 1e-300):.2e}"
        print(f"N={N}{' closed form' if cf else ' FFT'}: {np.median(ts[2:]):.3f} ms (min {min(ts[2:]):.3f}) per p=4 evolution + <Q>{msg}", flush=True)
