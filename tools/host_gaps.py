"""Per-step wall time of qva_evolve vs device time of the same step (events on the plan stream):
the difference is host-side latency (driver calls, scheduling) that leaves the GPU idle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wl = make_config("cfg4", n_override=n)
stream = torch.cuda.Stream()
P = Q.Plan(wl.dim, "x", n_qubits=n, stream=stream.cuda_stream)
P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
for _ in range(3):
    P.evolve(wl.theta)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
walls = []
ev[0].record(stream)
for i in range(20):
    t0 = time.perf_counter()
    P.evolve(wl.theta)
    f = P.expectation()
    walls.append((time.perf_counter() - t0) * 1e3)
    ev[i + 1].record(stream)
torch.cuda.synchronize()
dev = [ev[i].elapsed_time(ev[i + 1]) for i in range(20)]
print("wall  ", " ".join("%.1f" % w for w in walls))
print("device", " ".join("%.1f" % d for d in dev))
P.destroy()
