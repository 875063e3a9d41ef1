"""Repeated e2e steps (set_qualities_maxcut + evolve + expectation) with per-launch device times
(QVA_TRACE=1 on stderr); prints each step's wall time and its launches slower than 7 ms."""
import os, subprocess, sys
CHILD = r'''
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
cfg, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
wl = make_config(cfg, n_override=n)
P = Q.Plan(wl.dim, "x", n_qubits=n)
P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
P.set_profiling(True)
for i in range(steps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights); P.evolve(wl.theta); f = P.expectation()
    P.kernel_stats("tile")  # harvest events
    torch.cuda.synchronize()
    print("STEP %d %.1f" % (i, (time.perf_counter() - t0) * 1e3), file=sys.stderr, flush=True)
P.destroy()
'''
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = sys.argv[2] if len(sys.argv) > 2 else "30"
steps = sys.argv[3] if len(sys.argv) > 3 else "30"
r = subprocess.run([sys.executable, "-c", CHILD, cfg, n, steps], env=dict(os.environ, QVA_TRACE="1"),
                   capture_output=True, text=True)
cur = []
for l in r.stderr.splitlines():
    if l.startswith("[qva]"):
        cur.append(l)
    elif l.startswith("STEP"):
        slow = [x.split()[2] + ":" + x.split()[3] for x in cur if float(x.split()[3]) > 7.0]
        tot = sum(float(x.split()[3]) for x in cur)
        print(l, "device-sum %.1f" % tot, "slow:", " ".join(slow), flush=True)
        cur = []
    else:
        print(l)
