"""bench.py's e2e loop in isolation (torch stream plan, pinned inputs, CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg4")
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
P = Q.Plan(wl.dim, "x", n_qubits=30, stream=stream.cuda_stream)
P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
th = torch.from_numpy(np.ascontiguousarray(wl.theta)).pin_memory().numpy()
eu = torch.from_numpy(np.ascontiguousarray(wl.edges_u, np.int32)).pin_memory().numpy()
ev = torch.from_numpy(np.ascontiguousarray(wl.edges_v, np.int32)).pin_memory().numpy()
for _ in range(3):
    P.evolve(th); P.expectation()
for rep in range(3):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        P.set_qualities_maxcut(eu, ev); P.evolve(th); f = P.expectation()
    e1.record(stream); torch.cuda.synchronize()
    print("e2e ms/step %.2f" % (e0.elapsed_time(e1) / 5))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(5):
        P.evolve(th); f = P.expectation()
    e1.record(stream); torch.cuda.synchronize()
    print("value ms/step %.2f" % (e0.elapsed_time(e1) / 5))
P.destroy()
