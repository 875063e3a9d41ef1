"""The world > 1 code path of libqva, executed: 2 and 4 processes on ONE B200 (`-m gpu`).

Each process is one rank of a real multi-process plan (qva_plan_create_ex with world = G), so
every real-rank branch runs: the IPC-handle all-gather and min-vote at plan creation, the pass
stores into the peers' IPC-mapped buffers (COMM-psi exchange fused into the preceding pass,
PAPER.md:356-370), the barrier after it, the <Q> / batch all-reduces (COMM-grad_f,
PAPER.md:374-389), the circulant row/column transposes fused into the FFT pass stores, the
row-partitioned sparse mixer whose SpMV reads remote columns from the peers' IPC-mapped Taylor
buffers (the paper's distributed SpMV), the QAOAz mixer on a sharded state
(pair terms touching a rank qubit read the partner's IPC-mapped buffer), and -- with
QVA_FUSE_EXCHANGE=0 --
the send/recv exchange, transpose and term-gather fallbacks.  NCCL refuses two
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

    # ---- generic sparse mixer with W partitioned by rows (the paper's distributed SpMV) ----
    def rows_csr(W, lo, hi):
        rp, cols, vals = [0], [], []
        for r in range(lo, hi):
            nz = np.nonzero(W[r])[0]
            cols += list(nz)
            vals += list(W[r, nz])
            rp.append(len(cols))
        return np.array(rp, np.int64), np.array(cols, np.int32), np.array(vals, np.float64)

    N4 = 1000  # not a power of two: the partition remainder goes to the lowest ranks (R16)
    rng = np.random.default_rng(4242)
    W = np.where(rng.uniform(size=(N4, N4)) < 0.01, rng.uniform(-1, 1, (N4, N4)), 0.0)
    W = np.triu(W, 1)
    W = W + W.T
    q4 = rng.standard_normal(N4)
    th4 = rng.uniform(0, math.pi, 4)
    ref4 = O.evolve_sparse_dense(q4, W, th4)
    with Q.Plan(N4, "sparse", rank=rank, world=world, transport=T) as P:
        ln, off = P.get_partition()
        rp, cc, vv = rows_csr(W, off, off + ln)
        P.set_sparse_mixer_rows(rp, cc, vv, row_offset=off)
        res["s_peer"] = P.query("sparse_peer")
        P.set_qualities(q4[off:off + ln], offset=off)
        P.evolve(th4)
        res["s_damp"] = _amp_close(P.get_state(), ref4[off:off + ln])
        _f_close(P.expectation(), O.expectation(ref4, q4), O.expectation(ref4, np.abs(q4)))
    # the hypercube (sum_j X_j) as a row-partitioned CSR equals the X mixer (P12 cross-check)
    n5 = 12
    X = O.dense_sum_x(n5)
    q5 = O.maxcut_q(n5, *random_regular_graph(n5, 3, rng))
    th5 = rng.uniform(0, math.pi, 4)
    with Q.Plan(1 << n5, "sparse", rank=rank, world=world, transport=T) as P:
        ln, off = P.get_partition()
        rp, cc, vv = rows_csr(X, off, off + ln)
        P.set_sparse_mixer_rows(rp, cc, None, row_offset=off)
        P.set_qualities(q5[off:off + ln], offset=off)
        P.evolve(th5)
        _amp_close(P.get_state(), O.evolve_x(n5, q5, th5)[off:off + ln])

    # ---- QAOAz (parity mixer) on a sharded state: windows of local bits as tile passes, every pair
    # term touching a rank qubit as a peer pass reading the partner rank's IPC-mapped buffer ----
    n6 = 16
    rng = np.random.default_rng(606)
    u6, v6 = random_regular_graph(n6, 3, rng)
    q6 = O.maxcut_q(n6, u6, v6)
    th6 = rng.uniform(0, math.pi, 4)
    psi06 = np.zeros(1 << n6, np.complex128)
    idx = [x for x in range(1 << n6) if bin(x).count("1") == 8][:200]
    psi06[idx] = rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))
    psi06 /= np.linalg.norm(psi06)
    for seq in (list(range(n6)), [15, 0, 7, 14, 3, 9, 12, 1, 13, 5]):
        ref6 = O.evolve_parity(n6, q6, seq, th6, psi06)
        with Q.Plan(1 << n6, "parity", n_qubits=n6, rank=rank, world=world, transport=T) as P:
            ln, off = P.get_partition()
            P.set_parity_mixer(seq)
            P.set_qualities_maxcut(u6, v6)
            P.set_initial_state(psi06[off:off + ln], offset=off)
            P.evolve(th6)
            _amp_close(P.get_state(), ref6[off:off + ln])
            _f_close(P.expectation(), O.expectation(ref6, q6), O.expectation(ref6, np.abs(q6)))
            P.set_qualities(q6[off:off + ln], offset=off)  # stored q
            P.evolve(th6)
            _amp_close(P.get_state(), ref6[off:off + ln])
            P.reset_state()
            P.apply_mixer(0.41)  # step-level mixer on the sharded state
            _amp_close(P.get_state(), O.mixer_parity(psi06.copy(), seq, 0.41)[off:off + ln])

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
    # the K_N closed form on the same row-sharded state: one 16-B all-reduce of sum(psi) per layer
    with Q.Plan(wl.dim, "circulant", rank=rank, world=world, transport=T, complete_closed_form=True) as P:
        ln, off = P.get_partition()
        P.set_qualities(wl.q[off:off + ln], offset=off)
        P.set_circulant_eigenvalues_const(wl.lam0, wl.lam_rest)
        P.evolve(wl.theta)
        _amp_close(P.get_state(), ref3[off:off + ln])
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
        assert out[r]["s_peer"] == (1 if fuse else 0), out[r]
