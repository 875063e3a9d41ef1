"""ctypes wrapper around oracle/qva_oracle.c plus the small dense (numpy/scipy) oracles.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Citations are to
/root/reference/PAPER.md line numbers; readings R1..R22 are in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qva_oracle.c")
_LIB = os.path.join(_HERE, "libqva_oracle.so")

__all__ = [
    "build_oracle", "lib", "num_threads", "set_num_threads", "maxcut_q", "init_uniform", "phase", "mixer_x",
    "mixer_circulant_dense", "mixer_complete", "expectation", "norm2", "probabilities",
    "evolve_x", "evolve_complete", "evolve_circulant_dense", "evolve_circulant_fft", "mixer_circulant_fft",
    "lightcone_maxcut",
    "dense_sum_x", "mixer_sparse_dense", "evolve_sparse_dense", "c128",
    "mixer_parity", "evolve_parity", "parity_pairs",
    "maxcut_q_at", "kperm_count", "kperm_unrank", "kperm_cost", "kperm_qualities",
    "maxcut_term_q", "evolve_ex",
]


def build_oracle(force: bool = False) -> str:
    """Compile the C oracle (plain -O2, no fast-math; OpenMP only splits independent loops)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


@lru_cache(maxsize=1)
def lib():
    build_oracle()
    L = ctypes.CDLL(_LIB)
    d, i, u64 = ctypes.c_double, ctypes.c_int, ctypes.c_uint64
    P = ctypes.c_void_p
    L.or_num_threads.restype = i
    L.or_set_num_threads.argtypes = [i]
    L.or_maxcut_q.argtypes = [i, i, P, P, P, P]
    L.or_init_uniform.argtypes = [u64, P]
    L.or_phase.argtypes = [u64, P, P, d]
    L.or_mixer_x.argtypes = [i, P, d]
    L.or_mixer_circulant_dense.argtypes = [u64, P, P, d]
    L.or_mixer_complete.argtypes = [u64, P, d, d, d]
    L.or_expectation.argtypes = [u64, P, P]
    L.or_expectation.restype = d
    L.or_norm2.argtypes = [u64, P]
    L.or_norm2.restype = d
    L.or_probabilities.argtypes = [u64, P, P]
    L.or_evolve_x.argtypes = [i, P, P, P, i]
    L.or_evolve_complete.argtypes = [u64, P, P, P, i, d, d]
    L.or_evolve_circulant_dense.argtypes = [u64, P, P, P, P, i]
    L.or_mixer_parity.argtypes = [i, P, P, i, d]
    L.or_evolve_parity.argtypes = [i, P, P, P, i, P, i]
    L.or_lightcone_maxcut.argtypes = [i, i, P, P, P, P, i, i, P]
    L.or_lightcone_maxcut.restype = d
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def c128(psi) -> np.ndarray:
    a = np.ascontiguousarray(psi, dtype=np.complex128)
    return a


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the oracle's loops (timing only; results do not depend on it)."""
    lib().or_set_num_threads(int(n))


def maxcut_q(n: int, u, v, w=None) -> np.ndarray:
    """q_x = -cut_w(x) (PAPER.md:721-726 Eq. maxcut-cost, cfg sign, R10)."""
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    q = np.empty(1 << n, np.float64)
    wp = None
    if w is not None:
        w = np.ascontiguousarray(w, np.float64)
        wp = _ptr(w)
    lib().or_maxcut_q(n, len(u), _ptr(u), _ptr(v), wp, _ptr(q))
    return q


def maxcut_q_at(u, v, w, xs) -> np.ndarray:
    """q_x = -cut_w(x) at the given indices only (R10; vertex j = bit j of x, R8), for samples of
    states too large to enumerate.  Edge order summation, like maxcut_q."""
    out = []
    for x in xs:
        x = int(x)
        c = 0.0
        for k in range(len(u)):
            if ((x >> int(u[k])) ^ (x >> int(v[k]))) & 1:
                c += 1.0 if w is None else float(w[k])
        out.append(-c)
    return np.array(out, np.float64)


def init_uniform(N: int) -> np.ndarray:
    psi = np.empty(N, np.complex128)
    lib().or_init_uniform(N, _ptr(psi))
    return psi


def phase(psi: np.ndarray, q: np.ndarray, gamma: float) -> np.ndarray:
    """In place; returns psi.  PAPER.md:152-155, :307-313."""
    assert psi.dtype == np.complex128 and psi.flags.c_contiguous
    q = np.ascontiguousarray(q, np.float64)
    lib().or_phase(len(psi), _ptr(psi), _ptr(q), float(gamma))
    return psi


def mixer_x(psi: np.ndarray, beta: float) -> np.ndarray:
    """In place; PAPER.md:159-171 (R1: W = sum_j X_j)."""
    n = int(len(psi)).bit_length() - 1
    assert (1 << n) == len(psi)
    lib().or_mixer_x(n, _ptr(psi), float(beta))
    return psi


def mixer_circulant_dense(psi: np.ndarray, lam: np.ndarray, beta: float) -> np.ndarray:
    """In place; O(N^2) definition of F^-1 diag(e^{-i beta lam}) F (R3, R4)."""
    lam = np.ascontiguousarray(lam, np.float64)
    lib().or_mixer_circulant_dense(len(psi), _ptr(psi), _ptr(lam), float(beta))
    return psi


def mixer_complete(psi: np.ndarray, beta: float, lam0: float, lam_rest: float) -> np.ndarray:
    """In place; closed form for lambda = (lam0, c, ..., c) (R5)."""
    lib().or_mixer_complete(len(psi), _ptr(psi), float(beta), float(lam0), float(lam_rest))
    return psi


def expectation(psi: np.ndarray, q: np.ndarray) -> float:
    q = np.ascontiguousarray(q, np.float64)
    return float(lib().or_expectation(len(psi), _ptr(psi), _ptr(q)))


def norm2(psi: np.ndarray) -> float:
    return float(lib().or_norm2(len(psi), _ptr(psi)))


def probabilities(psi: np.ndarray) -> np.ndarray:
    out = np.empty(len(psi), np.float64)
    lib().or_probabilities(len(psi), _ptr(psi), _ptr(out))
    return out


def evolve_x(n: int, q: np.ndarray, theta, psi0: np.ndarray | None = None) -> np.ndarray:
    """QAOA state.  theta = [g1, b1, ...] (R7)."""
    theta = np.ascontiguousarray(theta, np.float64)
    p = len(theta) // 2
    psi = init_uniform(1 << n) if psi0 is None else np.array(psi0, np.complex128, copy=True)
    q = np.ascontiguousarray(q, np.float64)
    lib().or_evolve_x(n, _ptr(psi), _ptr(q), _ptr(theta), p)
    return psi


def evolve_complete(q: np.ndarray, theta, lam0: float, lam_rest: float,
                    psi0: np.ndarray | None = None) -> np.ndarray:
    """QWOA state with the complete-graph-family spectrum (R5, R20)."""
    theta = np.ascontiguousarray(theta, np.float64)
    N = len(q)
    psi = init_uniform(N) if psi0 is None else np.array(psi0, np.complex128, copy=True)
    q = np.ascontiguousarray(q, np.float64)
    lib().or_evolve_complete(N, _ptr(psi), _ptr(q), _ptr(theta), len(theta) // 2,
                             float(lam0), float(lam_rest))
    return psi


def evolve_circulant_dense(q: np.ndarray, lam: np.ndarray, theta,
                           psi0: np.ndarray | None = None) -> np.ndarray:
    theta = np.ascontiguousarray(theta, np.float64)
    N = len(q)
    psi = init_uniform(N) if psi0 is None else np.array(psi0, np.complex128, copy=True)
    q = np.ascontiguousarray(q, np.float64)
    lam = np.ascontiguousarray(lam, np.float64)
    lib().or_evolve_circulant_dense(N, _ptr(psi), _ptr(q), _ptr(lam), _ptr(theta), len(theta) // 2)
    return psi


def mixer_circulant_fft(psi: np.ndarray, lam: np.ndarray, beta: float) -> np.ndarray:
    """F^-1 diag(e^{-i beta lam}) F by the FFT the paper names for circulant mixers
    (Sec. 3; readings R3, R4: numpy's forward-DFT bin order).  Library
    primitive: numpy.fft (pocketfft).  Returns a new array."""
    lam = np.asarray(lam, np.float64)
    return np.fft.ifft(np.exp(-1j * beta * lam) * np.fft.fft(psi))


def evolve_circulant_fft(q: np.ndarray, lam: np.ndarray, theta,
                         psi0: np.ndarray | None = None) -> np.ndarray:
    """QWOA state prod_k U_M(beta_k) U_Q(gamma_k) |psi0> (PAPER.md:298 Eq. qwoa; theta layout
    R7) with the circulant mixer through mixer_circulant_fft: the large-N twin of
    evolve_circulant_dense (same loop; pinned against it in tests/test_oracle_pins.py P20)."""
    theta = np.asarray(theta, np.float64)
    N = len(q)
    psi = init_uniform(N) if psi0 is None else np.array(psi0, np.complex128, copy=True)
    for k in range(len(theta) // 2):
        phase(psi, q, float(theta[2 * k]))
        psi = np.ascontiguousarray(mixer_circulant_fft(psi, lam, float(theta[2 * k + 1])), np.complex128)
    return psi


def parity_pairs(seq):
    """(B_odd, B_even, B_last) qubit pairs of the QAOAz mixer over the ordered subsequence seq
    (PAPER.md:213-248 Eq. parity_terms; reading R19: no wrap in B_even, B_last = (s_{K-1}, s_0)
    iff K is odd)."""
    K = len(seq)
    odd = [(seq[m], seq[m + 1]) for m in range(0, K - 1, 2)]
    even = [(seq[m], seq[m + 1]) for m in range(1, K - 1, 2)]
    last = [(seq[K - 1], seq[0])] if K >= 3 and K % 2 == 1 else []
    return odd, even, last


def mixer_parity(psi: np.ndarray, seq, t: float) -> np.ndarray:
    """In place; U_parity(t) = e^{-itB_last} e^{-itB_even} e^{-itB_odd} (PAPER.md Eq. qaoaz_mixers)."""
    n = int(len(psi)).bit_length() - 1
    sq = np.ascontiguousarray(seq, np.int32)
    lib().or_mixer_parity(n, _ptr(psi), _ptr(sq), len(sq), float(t))
    return psi


def evolve_parity(n: int, q: np.ndarray, seq, theta, psi0: np.ndarray) -> np.ndarray:
    """QAOAz state (PAPER.md Eq. qaoaz) from a given (parity-constrained) initial state."""
    theta = np.ascontiguousarray(theta, np.float64)
    psi = np.array(psi0, np.complex128, copy=True)
    q = np.ascontiguousarray(q, np.float64)
    sq = np.ascontiguousarray(seq, np.int32)
    lib().or_evolve_parity(n, _ptr(psi), _ptr(q), _ptr(sq), len(sq), _ptr(theta), len(theta) // 2)
    return psi


def lightcone_maxcut(n: int, u, v, w, theta, max_qubits: int = 28):
    """Exact <Q> for q = -cut_w by per-edge light-cone simulation.  Returns (value, cone_sizes)."""
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    theta = np.ascontiguousarray(theta, np.float64)
    sizes = np.zeros(len(u), np.int32)
    wp = None
    if w is not None:
        w = np.ascontiguousarray(w, np.float64)
        wp = _ptr(w)
    val = lib().or_lightcone_maxcut(n, len(u), _ptr(u), _ptr(v), wp, _ptr(theta), len(theta) // 2,
                                    max_qubits, _ptr(sizes))
    return float(val), sizes


# ---------------------------------------------------------------------------------------
# Dense small-N oracles (library primitives: scipy.linalg.expm, numpy matmul).
# ---------------------------------------------------------------------------------------

def dense_sum_x(n: int) -> np.ndarray:
    """W = sum_j X_j as a dense real matrix (hypercube adjacency)."""
    N = 1 << n
    W = np.zeros((N, N))
    for j in range(n):
        idx = np.arange(N)
        W[idx, idx ^ (1 << j)] = 1.0
    return W


def mixer_sparse_dense(psi: np.ndarray, W_dense: np.ndarray, beta: float) -> np.ndarray:
    """exp(-i beta W) psi by scipy's dense expm -- the definition of the sparse mixer's
    result (PAPER.md:72-77 Eq. 4, :333).  Small N only."""
    from scipy.linalg import expm
    return expm(-1j * beta * np.asarray(W_dense, np.complex128)) @ psi


def evolve_sparse_dense(q: np.ndarray, W_dense: np.ndarray, theta,
                        psi0: np.ndarray | None = None) -> np.ndarray:
    """Generic QVA (Eq. 1) with phase U_Q and mixer exp(-i beta W) (dense)."""
    N = len(q)
    psi = init_uniform(N) if psi0 is None else np.array(psi0, np.complex128, copy=True)
    for k in range(len(theta) // 2):
        phase(psi, q, theta[2 * k])
        psi = np.ascontiguousarray(mixer_sparse_dense(psi, W_dense, theta[2 * k + 1]))
    return psi


# ---------------------------------------------------------------------------------------
# Permutation-encoded subspaces (QWOA).
# A solution s is a k-permutation of the m elements zeta = {0..m-1}; the
# indexed state |i> holds the i-th k-permutation in lexicographic order (reading R23: the
# indexing id_chi of Eq. qwoa_index is the Lehmer code / factorial number system).
# ---------------------------------------------------------------------------------------

def kperm_count(m: int, k: int) -> int:
    """|S'| = m! / (m - k)! (number of k-permutations of m elements)."""
    return math.perm(m, k)


def kperm_unrank(m: int, k: int, r: int) -> list:
    """The r-th k-permutation of range(m) in lexicographic order: digit a of the mixed-radix
    (Lehmer) code of r is r // ((m-a-1)!/(m-k)!), and it picks that many-th smallest unused
    element (R23)."""
    avail = list(range(m))
    out = []
    for a in range(k):
        c = math.perm(m - a - 1, k - a - 1)
        d, r = divmod(r, c)
        out.append(avail.pop(d))
    return out


def kperm_cost(pi, F, D, C=None) -> float:
    """C(s) = sum_a ( C[a, s_a] + sum_b F[a, b] D[s_a, s_b] ) (reading R24: the quadratic-
    assignment form; TSP is F = the directed cycle).  Summed in this order, a-major."""
    k = len(pi)
    s = 0.0
    for a in range(k):
        if C is not None:
            s += float(C[a][pi[a]])
        for b in range(k):
            s += float(F[a][b]) * float(D[pi[a]][pi[b]])
    return s


def kperm_qualities(m: int, k: int, F, D, C=None, ranks=None) -> np.ndarray:
    """q_i = C(s_i) for every rank i (or the given ranks): diag(Q) of the permutation subspace
    ("diag(Q) = C(s_i)").  Plain loops: small subspaces / samples only."""
    if ranks is None:
        ranks = range(kperm_count(m, k))
    return np.array([kperm_cost(kperm_unrank(m, k, int(r)), F, D, C) for r in ranks], np.float64)


# ---------------------------------------------------------------------------------------
# Extended QAOA (Eqs. phase_shift_qaoa_ex / qaoa_ex).
# ---------------------------------------------------------------------------------------

def maxcut_term_q(n: int, u: int, v: int, w: float = 1.0) -> np.ndarray:
    """Diagonal of one summation term of the max-cut quality (reading R25): Sigma_e(x) =
    -w_e [x_u != x_v], so that sum_e Sigma_e = q = -cut_w (R10)."""
    x = np.arange(1 << n, dtype=np.int64)
    return -float(w) * (((x >> u) ^ (x >> v)) & 1).astype(np.float64)


def evolve_ex(n: int, u, v, w, theta) -> np.ndarray:
    """ex-QAOA state (PAPER.md Eq. qaoa_ex): theta = per layer [gamma_{i,1..m}, t_i]
    (|theta| = (1 + m) D); layer i applies prod_e exp(-i gamma_{i,e} Sigma_e)
    (Eq. phase_shift_qaoa_ex: the terms commute) then U_X(t_i); layer 1 acts first (R6)."""
    m = len(u)
    theta = np.asarray(theta, np.float64)
    assert theta.size % (m + 1) == 0
    p = theta.size // (m + 1)
    psi = init_uniform(1 << n)
    for i in range(p):
        th = theta[i * (m + 1):(i + 1) * (m + 1)]
        for e in range(m):
            phase(psi, maxcut_term_q(n, int(u[e]), int(v[e]), 1.0 if w is None else float(w[e])), th[e])
        mixer_x(psi, th[m])
    return psi
