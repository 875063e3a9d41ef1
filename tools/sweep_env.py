"""Per-pass device times for the cfg4 recipe at n qubits under env settings: sweep_env.py n VAR=a,b,c"""
import os, subprocess, sys
CHILD = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
n = int(sys.argv[1])
wl = make_config(os.environ.get("QVA_SWEEP_CFG", "cfg4"), n_override=n)
with Q.Plan(wl.dim, "x", n_qubits=n) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    P.evolve(wl.theta); P.evolve(wl.theta)
    P.set_profiling(True); P.reset_kernel_stats()
    for _ in range(3): P.evolve(wl.theta)
    k = P.kernel_stats("tile")
    f = P.expectation()
print("ms/evolve(tile) %.2f f=%.12f" % (k["ms"] / 3, f), flush=True)
'''
n = sys.argv[1]
var, vals = sys.argv[2].split("=")
for v in vals.split(","):
    r = subprocess.run([sys.executable, "-c", CHILD, n], env=dict(os.environ, **{var: v}, QVA_TRACE="1"),
                       capture_output=True, text=True)
    tr = [l.split()[3] for l in r.stderr.splitlines() if l.startswith("[qva] class 0")]
    npass = int(os.environ.get("QVA_SWEEP_PASSES", "7"))
    print(var, v, r.stdout.strip() or r.stderr[-1500:], "passes:", " ".join(tr[-npass:]), flush=True)
