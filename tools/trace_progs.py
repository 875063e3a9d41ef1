"""Which tile-pass programs the schedules use (QVA_TRACE=2 prints one line per pass)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
for n, G, p in [(16, 1, 3), (20, 1, 3), (24, 4, 2), (26, 2, 3), (14, 1, 1)]:
    wl = make_config("cfg4", n_override=n)
    print(f"== n={n} G={G} p={p}", file=sys.stderr, flush=True)
    with Q.Plan(1 << n, "x", n_qubits=n, virtual_shards=G) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
        P.evolve(wl.theta[:2 * p])
