"""The world > 1 code path of libqva, executed: 2 and 4 processes on ONE B200 (`-m gpu`).

Each process is one rank of a real multi-process plan (qva_plan_create_ex with world = G), so
every real-rank branch runs: the IPC-handle all-gather and min-vote at plan creation, the pass
stores into the peers' IPC-mapped buffers (COMM-psi exchange fused into the preceding pass,
PAPER.md:356-370), the barrier after it, the <Q> / batch all-reduces (COMM-grad_f,
PAPER.md:374-389), the circulant row/column transposes fused into the FFT pass stores, and --
with QVA_FUSE_EXCHANGE=0 -- the send/recv exchange and transpose fallbacks.  NCCL refuses two
ranks on one device, so the plan's few collectives run over a host transport (torch gloo,
TorchHostTransport); the data path stays device-to-device through CUDA IPC.  No kernel waits on
another rank's kernel (every cross-rank ordering is a host-side barrier after a stream
synchronise), so the ranks may time-slice the GPU in any order.

Every rank compares its own partition (Eqs. local_i / offset) element by
element with the CPU oracle, at the north_star tolerances.
"""
import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
F_TOL = 1e-9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fuse, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["QVA_FUSE_EXCHANGE"] = "1" if fuse else "0"
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, "ok", _rank_checks(rank, world)))
    except Exception:
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(world, fuse):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fuse, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, st, res = q.get(timeout=600)
            assert st == "ok", f"rank {r}:\n{res}"
            out[r] = res
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return out


def _amp_close(got, ref):
    d = float(np.max(np.abs(got - ref))) if len(ref) else 0.0
    assert d <= AMP_TOL, d
    return d


def _f_close(got, ref, scale=None):
    s = max(abs(ref), scale or 0.0, 1e-300)
    assert abs(got - ref) <= F_TOL * s, (got, ref)


def _rank_checks(rank, world):
    import paper_2110_03963_b200 as Q
    import oracle as O
    from qva_inputs import random_regular_graph, make_config, fd_batch_thetas

    T = Q.TorchHostTransport()
    res = {}

    # ---- X mixer, sharded state (COMM-psi): n = 18, g = log2(world) global qubits ----
    n, p = 18, 3
    rng = np.random.default_rng(1000 + n)
    u, v = random_regular_graph(n, 4, rng)
    w = rng.uniform(0, 1, len(u))
    theta = rng.uniform(0, math.pi, 2 * p)
    q = O.maxcut_q(n, u, v, w)
    ref = O.evolve_x(n, q, theta)
    with Q.Plan(1 << n, "x", n_qubits=n, rank=rank, world=world, transport=T, max_batch=4) as P:
        assert P.query("host_transport") == 1 and P.query("shards") == world
        res["x_fused"] = P.query("fused_exchange")
        ln, off = P.get_partition()
        assert ln == (1 << n) // world and off == rank * ln
        P.set_qualities(q[off:off + ln], offset=off)     # stored q: layout-B copy built by the exchange
        P.evolve(theta)
        _f_close(P.expectation(), O.expectation(ref, q))
        res["x_damp"] = _amp_close(P.get_state(), ref[off:off + ln])
        np.testing.assert_allclose(P.get_probabilities(), np.abs(ref[off:off + ln]) ** 2, atol=1e-12)
        P.set_qualities_maxcut(u, v, w)                  # generated q: rank bits are tile constants
        P.evolve(theta)
        _amp_close(P.get_state(), ref[off:off + ln])
        _f_close(P.expectation(), O.expectation(ref, q))
        # step-level phase / mixer on the sharded state (mixer: exchange + rotation)
        P.reset_state()
        P.apply_phase(0.5)
        P.apply_mixer(1.3)
        r2 = O.init_uniform(1 << n)
        O.phase(r2, q, 0.5)
        O.mixer_x(r2, 1.3)
        _amp_close(P.get_state(), r2[off:off + ln])
        # sharded batch: each member's partial <Q> sums over ranks (all-reduce of B values)
        th = rng.uniform(0, math.pi, (3, 2 * p))
        f = P.evolve_batch(th)
        for b in range(3):
            _f_close(f[b], O.expectation(O.evolve_x(n, q, th[b]), q))
        # a non-uniform initial state, uploaded per partition
        psi0 = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        psi0 /= np.linalg.norm(psi0)
        P.set_initial_state(psi0[off:off + ln], offset=off)
        P.evolve(theta)
        _amp_close(P.get_state(), O.evolve_x(n, q, theta, psi0=psi0)[off:off + ln])

    # ---- replicated batch (COMM-grad_f): members split over ranks, f all-reduced ----
    n2, p2 = 14, 2
    rng = np.random.default_rng(77)
    u2, v2 = random_regular_graph(n2, 3, rng)
    q2 = O.maxcut_q(n2, u2, v2)
    th0 = rng.uniform(0, math.pi, 2 * p2)
    ths = fd_batch_thetas(th0, 1e-6)
    with Q.Plan(1 << n2, "x", n_qubits=n2, rank=rank, world=world, transport=T, replicated=True,
                max_batch=len(ths)) as P:
        P.set_qualities_maxcut(u2, v2)
        f = P.evolve_batch(ths)
        for b in range(len(ths)):
            _f_close(f[b], O.expectation(O.evolve_x(n2, q2, ths[b]), q2))

    # ---- circulant (QWOA) sharded by rows: cfg3, N = 10!, two transposes per layer (C5) ----
    wl = make_config("cfg3")
    ref3 = O.evolve_complete(wl.q, wl.theta, wl.lam0, wl.lam_rest)
    with Q.Plan(wl.dim, "circulant", rank=rank, world=world, transport=T) as P:
        res["c_fused"] = P.query("fused_exchange")
        ln, off = P.get_partition()
        P.set_qualities(wl.q[off:off + ln], offset=off)
        P.set_circulant_eigenvalues_const(wl.lam0, wl.lam_rest)
        P.evolve(wl.theta)
        res["c_damp"] = _amp_close(P.get_state(), ref3[off:off + ln])
        _f_close(P.expectation(), O.expectation(ref3, wl.q), scale=float(np.sum(np.abs(ref3) ** 2 * np.abs(wl.q))))
    return res


@pytest.fixture(scope="module")
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("fuse", [True, False], ids=["ipc_peer_stores", "fallback_alltoall"])
def test_world_gt1_plans_on_one_gpu(_gpu, world, fuse):
    out = _run(world, fuse)
    for r in range(world):
        # the fused path must really be the one that ran (IPC mapping succeeded on every rank)
        assert out[r]["x_fused"] == (1 if fuse else 0), out[r]
        assert out[r]["c_fused"] == (1 if fuse else 0), out[r]
