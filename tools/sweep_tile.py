"""Time the X-mixer evolution (cfg4 recipe at n qubits) for several L2-prefetch distances.
Each setting runs in a fresh process (the knob is read at library load)."""
import os
import subprocess
import sys

CHILD = r'''
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
n = int(sys.argv[1]); reps = int(sys.argv[2])
wl = make_config("cfg4", n_override=n)
with Q.Plan(wl.dim, "x", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    for _ in range(2):
        P.evolve(wl.theta)
    P.set_profiling(True)
    P.reset_kernel_stats()
    t0 = time.perf_counter()
    for _ in range(reps):
        P.evolve(wl.theta)
    dt = (time.perf_counter() - t0) / reps
    k = P.kernel_stats("tile"); ms, launches, by = k["ms"], k["launches"], k["bytes"]
    f = P.expectation()
print(json.dumps({"prefetch": os.environ.get("QVA_PREFETCH"), "n": n, "ms_per_evolve": dt * 1e3,
                  "tile_ms_per_launch": ms / launches, "tile_GBps": by / (ms * 1e-3) / 1e9, "f": f}))
'''

n = sys.argv[1] if len(sys.argv) > 1 else "30"
reps = sys.argv[2] if len(sys.argv) > 2 else "5"
vals = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "4"]
for v in vals:
    env = dict(os.environ, QVA_PREFETCH=v)
    r = subprocess.run([sys.executable, "-c", CHILD, n, reps], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
