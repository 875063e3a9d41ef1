"""Where the host-q e2e step goes (cfg4, n=30): pinned-host q upload, first evolve after it
(classification, int8 encoding, consumer-order copies), steady evolve.  CUDA-synchronised wall times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg4")
stream = torch.cuda.Stream()
with Q.Plan(wl.dim, "x", n_qubits=wl.n_qubits, stream=stream.cuda_stream) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
    if os.environ.get("PROF"):
        P.set_profiling(True)   # with QVA_TRACE=1: per-launch device times on stderr
    qh = torch.empty(wl.dim, dtype=torch.float64, pin_memory=True)
    qn = qh.numpy()
    P.get_qualities(0, wl.dim, out=qn)
    src = torch.empty(wl.dim, dtype=torch.float64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        src.copy_(qh, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
        P.set_qualities(qn); t2 = time.perf_counter()
        P.evolve(wl.theta); f = P.expectation(); t3 = time.perf_counter()
        P.evolve(wl.theta); f = P.expectation(); t4 = time.perf_counter()
        print(f"torch H2D 8 GiB {1e3*(t1-t0):.1f} ms ({wl.dim*8/(t1-t0)/1e9:.1f} GB/s) | set_qualities {1e3*(t2-t1):.1f} ms | "
              f"first evolve {1e3*(t3-t2):.1f} ms | steady evolve {1e3*(t4-t3):.1f} ms", flush=True)
