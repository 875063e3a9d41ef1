"""Host time of each call of the e2e step (set_qualities_maxcut / evolve / expectation)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg4")
P = Q.Plan(wl.dim, "x", n_qubits=30)
P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
for _ in range(3):
    P.evolve(wl.theta); P.expectation()
rows = []
for i in range(15):
    t0 = time.perf_counter(); P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
    t1 = time.perf_counter(); P.evolve(wl.theta)
    t2 = time.perf_counter(); f = P.expectation()
    t3 = time.perf_counter()
    rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
for r in rows: print("set %.3f  evolve %.2f  expect %.3f" % r)
P.destroy()
