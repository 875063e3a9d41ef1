"""B200-native QVA state evolution (arXiv 2110.03963 hot path) -- Python binding.

Thin ctypes marshalling over libqva.so (include/qva.h).  Every step of the method runs in
the sm_100a kernels behind the C ABI; this module only converts arguments.  There is no
CPU fallback: the first call into the package without the built library raises ImportError.

Module-level functions carry the ABI names (qva_plan_create, qva_set_qualities, qva_evolve,
qva_expectation, qva_evolve_batch, ...); `Plan` is a convenience owner of one plan handle.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqva.so")

MIXER_X, MIXER_CIRCULANT, MIXER_SPARSE, MIXER_PARITY = 0, 1, 2, 3
_MIXERS = {"x": MIXER_X, "circulant": MIXER_CIRCULANT, "sparse": MIXER_SPARSE, "parity": MIXER_PARITY}
KERNEL_CLASSES = {"tile": 0, "small": 1, "fft_col": 2, "fft_row": 3, "spmv": 4, "reduce": 5,
                  "exchange": 6, "other": 7, "fft_inner": 8}


class QvaError(RuntimeError):
    def __init__(self, func: str, status: int, msg: str):
        super().__init__(f"{func}: {status_string(status)}: {msg}")
        self.status = status


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_uint64),
        ("n_qubits", ctypes.c_int32),
        ("mixer", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("device", ctypes.c_int32),
        ("virtual_shards", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("max_batch", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 7),
    ]


_AG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64)
_AR_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32)
_A2A_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64)


class Transport(ctypes.Structure):
    """qva_transport (include/qva.h): host collectives of a world > 1 plan."""
    _fields_ = [("ctx", ctypes.c_void_p), ("allgather", _AG_FN), ("allreduce_f64", _AR_FN), ("alltoall", _A2A_FN)]


class TorchHostTransport:
    """qva_transport over an initialised torch.distributed CPU process group (gloo): the plan's
    collectives (IPC-handle all-gather, min-vote, barrier, <Q> / batch all-reduce, fallback
    all-to-all) run as torch collectives on host tensors.  Plumbing only: no arithmetic of the
    method.  Keep the object alive as long as the plan (Plan does)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._torch, self._dist, self._group = torch, dist, group
        self.world = dist.get_world_size(group)

        def _view(addr, nbytes):
            return self._torch.frombuffer((ctypes.c_char * nbytes).from_address(addr), dtype=self._torch.uint8)

        def allgather(_ctx, inp, out, nbytes):
            try:
                src = _view(inp, nbytes).clone()
                dst = self._torch.empty(self.world * nbytes, dtype=self._torch.uint8)
                self._dist.all_gather_into_tensor(dst, src, group=self._group)
                ctypes.memmove(out, dst.data_ptr(), self.world * nbytes)
                return 0
            except Exception:
                return 1

        def allreduce(_ctx, vals, n, op):
            try:
                t = self._torch.frombuffer((ctypes.c_double * n).from_address(vals), dtype=self._torch.float64)
                ops = {0: self._dist.ReduceOp.SUM, 1: self._dist.ReduceOp.MAX, 2: self._dist.ReduceOp.MIN}
                self._dist.all_reduce(t, op=ops[int(op)], group=self._group)
                return 0
            except Exception:
                return 1

        def alltoall(_ctx, send, recv, chunk):
            try:
                src = _view(send, self.world * chunk).clone()
                dst = self._torch.empty(self.world * chunk, dtype=self._torch.uint8)
                self._dist.all_to_all_single(dst, src, group=self._group)
                ctypes.memmove(recv, dst.data_ptr(), self.world * chunk)
                return 0
            except Exception:
                return 1

        self._fns = (_AG_FN(allgather), _AR_FN(allreduce), _A2A_FN(alltoall))
        self.struct = Transport(None, *self._fns)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2110_03963_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, u64, i32, d = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double
    sig = {
        "qva_plan_create": [ctypes.POINTER(PlanDesc), ctypes.POINTER(P)],
        "qva_plan_create_ex": [ctypes.POINTER(PlanDesc), ctypes.POINTER(Transport), ctypes.POINTER(P)],
        "qva_plan_destroy": [P],
        "qva_plan_get_partition": [P, ctypes.POINTER(u64), ctypes.POINTER(u64)],
        "qva_partition": [u64, i32, i32, ctypes.POINTER(u64), ctypes.POINTER(u64)],
        "qva_set_qualities": [P, P, u64, u64],
        "qva_set_qualities_device": [P, P, u64, u64],
        "qva_set_qualities_maxcut": [P, i32, P, P, P],
        "qva_set_qualities_permutation": [P, i32, i32, P, P, P],
        "qva_get_qualities": [P, P, u64, u64],
        "qva_set_circulant_eigenvalues": [P, P, u64, u64],
        "qva_set_circulant_eigenvalues_const": [P, d, d],
        "qva_set_sparse_mixer": [P, P, P, P, u64],
        "qva_set_sparse_mixer_rows": [P, P, P, P, u64, u64, u64],
        "qva_set_parity_mixer": [P, P, i32],
        "qva_parity_schedule": [i32, P, i32, P, i32, ctypes.POINTER(i32)],
        "qva_set_initial_state": [P, P, u64, u64],
        "qva_clear_initial_state": [P],
        "qva_reset_state": [P],
        "qva_apply_phase": [P, d],
        "qva_apply_mixer": [P, d],
        "qva_evolve": [P, P, i32],
        "qva_expectation": [P, ctypes.POINTER(d)],
        "qva_norm2": [P, ctypes.POINTER(d)],
        "qva_get_state": [P, P, u64, u64],
        "qva_get_probabilities": [P, P, u64, u64],
        "qva_evolve_batch": [P, P, i32, i32, P],
        "qva_evolve_ex": [P, P, i32],
        "qva_evolve_ex_batch": [P, P, i32, i32, P],
        "qva_nccl_unique_id": [P],
        "qva_batch_partition": [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)],
        "qva_exchange_plan": [i32, i32, P, P],
        "qva_x_schedule": [i32, i32, P, i32, ctypes.POINTER(i32)],
        "qva_x_schedule_permuted": [i32, i32, P, i32, ctypes.POINTER(i32)],
        "qva_circulant_plan_shape": [ctypes.c_uint64, i32, i32, P],
        "qva_set_profiling": [P, i32],
        "qva_kernel_stats": [P, i32, ctypes.POINTER(d), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(d)],
        "qva_reset_kernel_stats": [P],
        "qva_launch_count": [P, ctypes.POINTER(ctypes.c_int64)],
        "qva_plan_query": [P, i32, ctypes.POINTER(ctypes.c_int64)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    for name in ("qva_status_string", "qva_last_error", "qva_version"):
        getattr(L, name).restype = ctypes.c_char_p
    L.qva_status_string.argtypes = [ctypes.c_int]
    return L


_L = None


def lib():
    """The loaded libqva.so (loaded on first use so the build module can run without it)."""
    global _L
    if _L is None:
        _L = _load()
    return _L


def status_string(s: int) -> str:
    return lib().qva_status_string(int(s)).decode()


def _call(name: str, *args):
    st = getattr(lib(), name)(*args)
    if st != 0:
        raise QvaError(name, st, lib().qva_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def qva_version() -> str:
    return lib().qva_version().decode()


def qva_partition(dim: int, world: int, rank: int):
    n, o = ctypes.c_uint64(), ctypes.c_uint64()
    _call("qva_partition", dim, world, rank, ctypes.byref(n), ctypes.byref(o))
    return n.value, o.value


def qva_batch_partition(B: int, world: int, rank: int):
    f, c = ctypes.c_int32(), ctypes.c_int32()
    _call("qva_batch_partition", B, world, rank, ctypes.byref(f), ctypes.byref(c))
    return f.value, c.value


def qva_x_schedule(n_local: int, p: int):
    """[(tile_set, n_rot_before_phase, has_phase, n_rot_after_phase)] of the X-mixer passes."""
    cap = 4 * (3 * p + 8)
    out = np.zeros(4 * cap, np.int32)
    n = ctypes.c_int32()
    _call("qva_x_schedule", n_local, p, _ptr(out), cap, ctypes.byref(n))
    return [tuple(int(v) for v in out[4 * i:4 * i + 4]) for i in range(n.value)]


def qva_x_schedule_permuted(n_local: int, p: int):
    """Per pass of the permuted single-shard schedule: dict(window, a1, a2, phase, expect, r1, r2,
    dims) with r1/r2 the logical-qubit masks rotated before/after the phase (include/qva.h)."""
    cap = 64 * (p + 1)
    out = np.zeros(8 * cap, np.int64)
    n = ctypes.c_int32()
    _call("qva_x_schedule_permuted", n_local, p, _ptr(out), cap, ctypes.byref(n))
    keys = ("window", "a1", "a2", "phase", "expect", "r1", "r2", "dims")
    return [dict(zip(keys, (int(x) for x in out[8 * i:8 * i + 8]))) for i in range(min(n.value, cap))]


def qva_parity_schedule(n: int, seq):
    """Window passes of the QAOAz parity mixer (host-only): list of (window bits, [(a, b), ...])."""
    sq = np.ascontiguousarray(seq, np.int32)
    cap = 4096
    out = np.zeros(cap, np.int32)
    nw = ctypes.c_int32()
    _call("qva_parity_schedule", int(n), _ptr(sq), len(sq), _ptr(out), cap, ctypes.byref(nw))
    res, pos = [], 0
    for _ in range(nw.value):
        w, npairs = int(out[pos]), int(out[pos + 1])
        bits = [int(b) for b in out[pos + 2:pos + 2 + w]]
        pr = out[pos + 2 + w:pos + 2 + w + 2 * npairs].reshape(-1, 2)
        res.append((bits, [(int(a), int(b)) for a, b in pr]))
        pos += 2 + w + 2 * npairs
    return res


def qva_circulant_plan_shape(dim: int, shards: int = 1, three_level: bool = False):
    """dict(kind, M, M1, M2, cw, rb, levels, Mi1, Mi2) of the circulant mixer's FFT plan (include/qva.h)."""
    out = np.zeros(9, np.int64)
    _call("qva_circulant_plan_shape", dim, shards, 1 if three_level else 0, _ptr(out))
    return dict(zip(("kind", "M", "M1", "M2", "cw", "rb", "levels", "Mi1", "Mi2"), (int(x) for x in out)))


def qva_exchange_plan(G: int, rank: int):
    """(peer_of_chunk[G], peer_chunk[G]) of the global<->local qubit swap (include/qva.h)."""
    peer = np.zeros(G, np.int32)
    pchunk = np.zeros(G, np.int32)
    _call("qva_exchange_plan", G, rank, _ptr(peer), _ptr(pchunk))
    return peer, pchunk


def qva_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _call("qva_nccl_unique_id", ctypes.cast(buf, ctypes.c_void_p))
    return buf.raw


def nccl_id_broadcast(group=None) -> bytes:
    """NCCL bootstrap over an initialised torch.distributed group (any backend): rank 0 creates
    the 128-byte ncclUniqueId with qva_nccl_unique_id, every rank receives it by a uint8
    broadcast.  Pass the result as Plan(..., nccl_id=...) on every rank."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(qva_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Plan:
    """Owns one qva_plan.  Method names follow the C ABI without the `qva_` prefix."""

    def __init__(self, dim: int, mixer: str = "x", n_qubits: int = -1, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, device: int = 0, virtual_shards: int = 1,
                 stream: Optional[int] = None, max_batch: int = 1, replicated: bool = False,
                 qgen_f64_always: bool = False, fft_three_level: bool = False,
                 peer_store_exchange: bool = False, transport: Optional[TorchHostTransport] = None,
                 complete_closed_form: bool = False):
        """transport: a TorchHostTransport (world > 1) to run the plan's collectives over a torch
        host process group instead of NCCL (include/qva.h qva_plan_create_ex)."""
        self._h = ctypes.c_void_p()
        self._transport = transport
        self._id_buf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        d = PlanDesc()
        d.dim = dim
        d.n_qubits = n_qubits
        d.mixer = _MIXERS[mixer] if isinstance(mixer, str) else int(mixer)
        d.rank = rank
        d.world = world
        d.nccl_unique_id = ctypes.cast(self._id_buf, ctypes.c_void_p) if self._id_buf is not None else None
        d.device = device
        d.virtual_shards = virtual_shards
        d.stream = stream
        d.max_batch = max_batch
        d.reserved[0] = 1 if replicated else 0
        d.reserved[1] = 1 if qgen_f64_always else 0
        d.reserved[2] = 1 if fft_three_level else 0
        d.reserved[3] = 1 if peer_store_exchange else 0
        d.reserved[4] = 1 if complete_closed_form else 0
        if transport is not None:
            _call("qva_plan_create_ex", ctypes.byref(d), ctypes.byref(transport.struct), ctypes.byref(self._h))
        else:
            _call("qva_plan_create", ctypes.byref(d), ctypes.byref(self._h))
        self.dim, self.mixer, self.world, self.rank = dim, mixer, world, rank

    # ---- lifecycle
    def destroy(self):
        if self._h:
            _call("qva_plan_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()

    def get_partition(self):
        n, o = ctypes.c_uint64(), ctypes.c_uint64()
        _call("qva_plan_get_partition", self._h, ctypes.byref(n), ctypes.byref(o))
        return n.value, o.value

    # ---- operators
    def set_qualities(self, q, offset: int = 0):
        q = _f64(q)
        _call("qva_set_qualities", self._h, _ptr(q), offset, len(q))

    def set_qualities_device(self, ptr: int, offset: int, count: int):
        _call("qva_set_qualities_device", self._h, ctypes.c_void_p(ptr), offset, count)

    def set_qualities_maxcut(self, u, v, w=None):
        u = np.ascontiguousarray(u, np.int32)
        v = np.ascontiguousarray(v, np.int32)
        w = None if w is None else _f64(w)
        _call("qva_set_qualities_maxcut", self._h, len(u), _ptr(u), _ptr(v), _ptr(w))
        self._n_edges = len(u)

    def set_qualities_permutation(self, m: int, k: int, F=None, D=None, lin=None):
        """q_i = C(s_i), s_i the i-th k-permutation of range(m) in lexicographic order,
        C(s) = sum_a (lin[a, s_a] + sum_b F[a, b] D[s_a, s_b]) (readings R23, R24); generated on
        the device.  F: (k, k), D: (m, m), lin: (k, m), each optional (D required with F)."""
        F = None if F is None else _f64(np.asarray(F, np.float64).reshape(k, k))
        D = None if D is None else _f64(np.asarray(D, np.float64).reshape(m, m))
        lin = None if lin is None else _f64(np.asarray(lin, np.float64).reshape(k, m))
        _call("qva_set_qualities_permutation", self._h, int(m), int(k), _ptr(F), _ptr(D), _ptr(lin))

    def get_qualities(self, offset: int = 0, count: Optional[int] = None, out: Optional[np.ndarray] = None):
        if count is None:
            n, o = self.get_partition()
            offset, count = o, n
        if out is None:
            out = np.empty(count, np.float64)
        _call("qva_get_qualities", self._h, _ptr(out), offset, count)
        return out

    def set_circulant_eigenvalues(self, lam, offset: int = 0):
        lam = _f64(lam)
        _call("qva_set_circulant_eigenvalues", self._h, _ptr(lam), offset, len(lam))

    def set_circulant_eigenvalues_const(self, lam0: float, c: float):
        _call("qva_set_circulant_eigenvalues_const", self._h, float(lam0), float(c))

    def set_sparse_mixer(self, row_ptr, col, val=None):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = None if val is None else _f64(val)
        _call("qva_set_sparse_mixer", self._h, _ptr(row_ptr), _ptr(col), _ptr(val), len(col))

    def set_sparse_mixer_rows(self, row_ptr, col, val=None, row_offset: int = 0):
        """This rank's rows of a row-partitioned W (world > 1; include/qva.h): local row_ptr,
        global column indices.  Collective."""
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = None if val is None else _f64(val)
        _call("qva_set_sparse_mixer_rows", self._h, _ptr(row_ptr), _ptr(col), _ptr(val), int(row_offset),
              len(row_ptr) - 1, len(col))

    def set_parity_mixer(self, qubits):
        """Ordered qubit subsequence of the QAOAz parity mixer (include/qva.h)."""
        s = np.ascontiguousarray(qubits, np.int32)
        _call("qva_set_parity_mixer", self._h, _ptr(s), len(s))

    def set_initial_state(self, psi, offset: int = 0):
        psi = np.ascontiguousarray(psi, np.complex128)
        _call("qva_set_initial_state", self._h, _ptr(psi), offset, len(psi))

    def clear_initial_state(self):
        _call("qva_clear_initial_state", self._h)

    # ---- evolution
    def reset_state(self):
        _call("qva_reset_state", self._h)

    def apply_phase(self, gamma: float):
        _call("qva_apply_phase", self._h, float(gamma))

    def apply_mixer(self, beta: float):
        _call("qva_apply_mixer", self._h, float(beta))

    def evolve(self, theta):
        theta = _f64(theta)
        _call("qva_evolve", self._h, _ptr(theta), len(theta) // 2)

    def expectation(self) -> float:
        out = ctypes.c_double()
        _call("qva_expectation", self._h, ctypes.byref(out))
        return out.value

    def norm2(self) -> float:
        out = ctypes.c_double()
        _call("qva_norm2", self._h, ctypes.byref(out))
        return out.value

    def get_state(self, offset: int = 0, count: Optional[int] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        if count is None:
            n, o = self.get_partition()
            offset, count = o, n
        if out is None:
            out = np.empty(count, np.complex128)
        _call("qva_get_state", self._h, _ptr(out), offset, count)
        return out

    def get_probabilities(self, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            n, o = self.get_partition()
            offset, count = o, n
        out = np.empty(count, np.float64)
        _call("qva_get_probabilities", self._h, _ptr(out), offset, count)
        return out

    def evolve_batch(self, thetas) -> np.ndarray:
        thetas = np.ascontiguousarray(thetas, np.float64)
        B, P2 = thetas.shape
        out = np.empty(B, np.float64)
        _call("qva_evolve_batch", self._h, _ptr(thetas), B, P2 // 2, _ptr(out))
        return out

    def evolve_ex(self, theta):
        """ex-QAOA (PAPER.md Eq. qaoa_ex, R25): theta = per layer [gamma_{i,1..m}, t_i] over the
        m edges of the max-cut graph set by set_qualities_maxcut."""
        theta = _f64(theta)
        m1 = getattr(self, "_n_edges", 0) + 1
        if theta.size % m1:
            raise ValueError(f"ex-QAOA theta length {theta.size} is not a multiple of m + 1 = {m1}")
        _call("qva_evolve_ex", self._h, _ptr(theta), theta.size // m1)

    def evolve_ex_batch(self, thetas) -> np.ndarray:
        thetas = np.ascontiguousarray(thetas, np.float64)
        B, T = thetas.shape
        m1 = getattr(self, "_n_edges", 0) + 1
        if T % m1:
            raise ValueError(f"ex-QAOA theta length {T} is not a multiple of m + 1 = {m1}")
        out = np.empty(B, np.float64)
        _call("qva_evolve_ex_batch", self._h, _ptr(thetas), B, T // m1, _ptr(out))
        return out

    # ---- introspection
    def set_profiling(self, on: bool = True):
        _call("qva_set_profiling", self._h, 1 if on else 0)

    def kernel_stats(self, which) -> dict:
        k = KERNEL_CLASSES[which] if isinstance(which, str) else int(which)
        ms, n, b = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _call("qva_kernel_stats", self._h, k, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b))
        return {"ms": ms.value, "launches": n.value, "bytes": b.value}

    def reset_kernel_stats(self):
        _call("qva_reset_kernel_stats", self._h)

    def query(self, what) -> int:
        """qva_plan_query: 'fused_exchange', 'shards', 'host_transport', 'world', 'rank', 'xfer_bytes' (0..5)."""
        keys = {"fused_exchange": 0, "shards": 1, "host_transport": 2, "world": 3, "rank": 4, "xfer_bytes": 5,
                "parity_tile": 6, "sparse_peer": 7}
        out = ctypes.c_int64()
        _call("qva_plan_query", self._h, keys.get(what, what), ctypes.byref(out))
        return out.value

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        _call("qva_launch_count", self._h, ctypes.byref(n))
        return n.value
