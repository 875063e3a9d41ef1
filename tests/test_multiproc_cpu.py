"""Multi-process host logic of the sharded path on CPU (torch.distributed, gloo, world_size 2/4).

The pool gives one GPU per call, so the cross-rank parts that do not need a device are tested
here with real processes (SURVEY §4 tier 3-4):
  * the NCCL-id bootstrap of the binding (rank 0 creates the 128-byte id, everyone receives it);
  * COMM-psi partition (Eqs. local_i / offset): disjoint cover of [0, N);
  * the global<->local qubit exchange plan of libqva (qva_exchange_plan), executed with
    torch all_to_all: afterwards every element sits where the g global index bits and the top
    g local bits are swapped (the layout the sharded schedule assumes), and a second exchange
    restores layout A;
  * the COMM-grad-f batch split: members split by qva_batch_partition,
    evaluated per rank (here by the CPU oracle, at n = 8, because this file runs without a
    GPU), zero-filled and sum-all-reduced, equal the serial evaluation.
The library's own world > 1 path (plan creation with world = 2/4, IPC peer stores, the
barrier, its batch and <Q> all-reduces, the send/recv fallbacks) runs in
tests/test_multiproc_gpu.py: real ranks as processes on one GPU over a gloo host transport.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = globals()[fn_name](rank, world)
        q.put((rank, "ok", res))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(fn_name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, st, res = q.get(timeout=240)
        assert st == "ok", res
        out[r] = res
    for p in procs:
        p.join(timeout=60)
    return out


# ----------------------------------------------------------------------------- workers
def _w_bootstrap(rank, world):
    import paper_2110_03963_b200 as Q
    return Q.nccl_id_broadcast()


def _w_partition(rank, world):
    import paper_2110_03963_b200 as Q
    N = 10 * 9 * 8 * 7 + 3  # not a multiple of world: exercises the remainder rule (R16)
    n, o = Q.qva_partition(N, world, rank)
    t = torch.tensor([n, o], dtype=torch.int64)
    g = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(g, t)
    return [tuple(x.tolist()) for x in g]


def _swap_bits(x, L, g):
    """index with the top g bits (rank bits, above L local bits) swapped with local bits L-g..L-1"""
    hi = x >> L
    mid = (x >> (L - g)) & ((1 << g) - 1)
    lo = x & ((1 << (L - g)) - 1)
    return (mid << L) | (hi << (L - g)) | lo


def _w_exchange(rank, world):
    import paper_2110_03963_b200 as Q
    g = world.bit_length() - 1
    L = 6
    C = (1 << L) // world
    local = torch.arange(rank << L, (rank + 1) << L, dtype=torch.int64)  # global indices (layout A)

    def exchange(buf):
        peer, pchunk = Q.qva_exchange_plan(world, rank)
        # chunk t goes to peer[t]; what arrives from peer[t] lands in chunk t
        # the library's grouped ncclSend/ncclRecv, here as gloo point-to-point pairs
        out = torch.zeros_like(buf)
        reqs, recvs = [], []
        for t in range(world):
            if peer[t] == rank:
                assert t == rank
                out[t * C:(t + 1) * C] = buf[t * C:(t + 1) * C]
                continue
            assert pchunk[t] == rank
            reqs.append(dist.isend(buf[t * C:(t + 1) * C].clone(), int(peer[t])))
            rbuf = torch.zeros(C, dtype=torch.int64)
            reqs.append(dist.irecv(rbuf, int(peer[t])))
            recvs.append((t, rbuf))
        for r in reqs:
            r.wait()
        for t, rbuf in recvs:
            out[t * C:(t + 1) * C] = rbuf
        return out

    b = exchange(local)
    # layout B: the element at (rank, local i) has global index swap(rank, i)
    want = torch.tensor([_swap_bits((rank << L) | i, L, g) for i in range(1 << L)], dtype=torch.int64)
    ok_b = bool(torch.equal(b, want))
    a = exchange(b)
    return ok_b, bool(torch.equal(a, local))


def _w_batch(rank, world):
    # host logic only (member partition + all-reduce of the members' values): libqva needs a GPU to
    # create a plan; the library's own sharded batch and its all-reduce run in
    # tests/test_multiproc_gpu.py (world = 2 / 4 plans on one B200, every member vs the oracle)
    import oracle as O
    import paper_2110_03963_b200 as Q
    rng = np.random.default_rng(7)
    n, p, B = 8, 2, 9
    q = rng.standard_normal(1 << n)
    thetas = rng.uniform(0, np.pi, (B, 2 * p))
    first, cnt = Q.qva_batch_partition(B, world, rank)
    f = torch.zeros(B, dtype=torch.float64)
    for b in range(first, first + cnt):
        f[b] = O.expectation(O.evolve_x(n, q, thetas[b]), q)
    dist.all_reduce(f)
    serial = [O.expectation(O.evolve_x(n, q, thetas[b]), q) for b in range(B)]
    return float(np.max(np.abs(f.numpy() - np.array(serial))))


# ----------------------------------------------------------------------------- tests
def test_nccl_id_bootstrap_gloo_world2():
    out = _run("_w_bootstrap", 2)
    assert len(out[0]) == 128 and out[0] == out[1]


@pytest.mark.parametrize("world", [2, 4])
def test_partition_covers_disjointly(world):
    parts = _run("_w_partition", world)[0]
    N = 10 * 9 * 8 * 7 + 3
    pos = 0
    for n, o in parts:
        assert o == pos
        pos += n
    assert pos == N
    assert max(n for n, _ in parts) - min(n for n, _ in parts) <= 1


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_plan_swaps_global_and_top_local_bits(world):
    out = _run("_w_exchange", world)
    for r in range(world):
        assert out[r] == (True, True), (r, out[r])


def test_batch_split_allreduce_equals_serial():
    out = _run("_w_batch", 2)
    assert out[0] <= 1e-15 and out[1] <= 1e-15
