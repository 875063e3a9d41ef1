"""Write tests/golden/*.json for the full-size configs.  Calls ONLY oracle/ (and the
seeded input module); no value here ever comes from the CUDA path.

  python -m oracle.make_golden [cfg4] [cfg5] [weak]

cfg4 (n=30, p=3): full-state oracle (16 GiB state + 8 GiB q in host RAM) -> <Q>, norm^2,
                  and amplitudes at 4096 seeded sample indices; plus the light-cone <Q>.
cfg5 (n=34, p=2): light-cone <Q> (exact reduction).
weak:             light-cone <Q> for the cfg5 family at n = 30, 31, 32, 33 (weak-scaling series).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

import oracle as O
from qva_inputs import make_config

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sample_indices(n: int, k: int = 4096, seed: int = 1234) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = np.unique(rng.integers(0, 1 << n, size=k, dtype=np.int64))
    # always include the extremes
    return np.unique(np.concatenate([idx, [0, 1, (1 << n) - 2, (1 << n) - 1]])).astype(np.int64)


def _dump(name, obj):
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, name), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name, flush=True)


def golden_cfg4():
    wl = make_config("cfg4")
    n = wl.n_qubits
    t0 = time.time()
    lc, sizes = O.lightcone_maxcut(n, wl.edges_u, wl.edges_v, wl.weights, wl.theta, max_qubits=30)
    t_lc = time.time() - t0
    print("cfg4 light-cone", lc, "max cone", sizes.max(), f"{t_lc:.1f}s", flush=True)
    t0 = time.time()
    q = O.maxcut_q(n, wl.edges_u, wl.edges_v, wl.weights)
    psi = O.evolve_x(n, q, wl.theta)
    f = O.expectation(psi, q)
    nrm = O.norm2(psi)
    t_full = time.time() - t0
    idx = sample_indices(n)
    amps = psi[idx]
    print("cfg4 full", f, nrm, f"{t_full:.1f}s", flush=True)
    _dump("cfg4_n30.json", {
        "source": "oracle/make_golden.py (oracle only); PAPER.md:185 Eq. qaoa, :53-60 Eq. 2",
        "config": "cfg4", "n": n, "p": wl.p, "theta": wl.theta.tolist(),
        "expectation_full_state": f, "expectation_lightcone": lc, "norm2": nrm,
        "cone_sizes": sizes.tolist(), "oracle_threads": O.num_threads(),
        "seconds_full_state": t_full, "seconds_lightcone": t_lc,
        "sample_index": idx.tolist(), "sample_re": amps.real.tolist(), "sample_im": amps.imag.tolist(),
    })


def golden_lightcone(name, n=None, fname=None):
    wl = make_config(name, n_override=n)
    t0 = time.time()
    lc, sizes = O.lightcone_maxcut(wl.n_qubits, wl.edges_u, wl.edges_v, wl.weights, wl.theta, max_qubits=30)
    dt = time.time() - t0
    print(name, wl.n_qubits, lc, sizes.max(), f"{dt:.1f}s", flush=True)
    _dump(fname, {
        "source": "oracle/make_golden.py light-cone mode (oracle only); PAPER.md:185, :53-60",
        "config": name, "n": wl.n_qubits, "p": wl.p, "theta": wl.theta.tolist(),
        "expectation_lightcone": lc, "cone_sizes": sizes.tolist(),
        "oracle_threads": O.num_threads(), "seconds": dt,
    })


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg5", "weak", "cfg4"]
    if "cfg5" in which:
        golden_lightcone("cfg5", None, "cfg5_n34.json")
    if "weak" in which:
        for n in (30, 31, 32, 33):
            golden_lightcone("cfg5", n, f"cfg5_n{n}.json")
    if "cfg4" in which:
        golden_cfg4()
