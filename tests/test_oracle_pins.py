"""Pins of the CPU oracle against things other than itself (`-m "not gpu"`).

Each test names the pin (P1..P15) and the passage it follows.
Independent sources: scipy.linalg.expm, numpy.fft, networkx.cut_size, closed forms,
special cases and worked examples from SPEC.md.
"""
import math

import networkx as nx
import numpy as np
import pytest
from scipy.linalg import circulant, expm

import oracle as O
from qva_inputs import make_config, random_regular_graph, erdos_renyi_graph, fd_batch_thetas


def _rand_state(N, rng):
    psi = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    return np.ascontiguousarray(psi / np.linalg.norm(psi))


# ---------------------------------------------------------------- qualities (Eq. 24) ----
@pytest.mark.parametrize("weighted", [False, True])
def test_maxcut_q_vs_networkx(weighted):
    """q_x = -cut_w(x) (R10) against networkx.cut_size on every x."""
    rng = np.random.default_rng(11)
    n = 7
    u, v = erdos_renyi_graph(n, 0.6, rng)
    w = rng.uniform(0, 1, len(u)) if weighted else None
    G = nx.Graph()
    G.add_nodes_from(range(n))
    for k in range(len(u)):
        G.add_edge(int(u[k]), int(v[k]), weight=float(w[k]) if weighted else 1.0)
    q = O.maxcut_q(n, u, v, w)
    for x in range(1 << n):
        S = [j for j in range(n) if (x >> j) & 1]
        ref = nx.cut_size(G, S, weight="weight")
        assert q[x] == pytest.approx(-ref, abs=1e-13)


@pytest.mark.parametrize("weighted", [False, True])
def test_maxcut_q_at_vs_networkx(weighted):
    """maxcut_q_at (sampled q for huge n) against networkx.cut_size at n = 33 sampled states."""
    rng = np.random.default_rng(12)
    n = 33
    u, v = erdos_renyi_graph(n, 0.15, rng)
    w = rng.uniform(0, 1, len(u)) if weighted else None
    G = nx.Graph()
    G.add_nodes_from(range(n))
    for k in range(len(u)):
        G.add_edge(int(u[k]), int(v[k]), weight=float(w[k]) if weighted else 1.0)
    xs = rng.integers(0, 1 << n, 20)
    q = O.maxcut_q_at(u, v, w, xs)
    for x, qv in zip(xs, q):
        S = [j for j in range(n) if (int(x) >> j) & 1]
        assert qv == pytest.approx(-nx.cut_size(G, S, weight="weight"), abs=1e-12)


def test_maxcut_q_single_edge_spec_example():
    """SPEC.md:446 single edge (0,1), n=2: equal-bit states are uncut -> q = -(0,1,1,0)."""
    q = O.maxcut_q(2, [0], [1])
    assert list(q) == [0.0, -1.0, -1.0, 0.0]


# ---------------------------------------------------------------- phase / expectation ----
def test_phase_spec_example():
    """P15: SPEC.md:129-131: gamma=pi, o=(0,1,2,3), uniform_4 -> (1,-1,1,-1)/2."""
    psi = O.init_uniform(4)
    O.phase(psi, np.array([0.0, 1, 2, 3]), math.pi)
    np.testing.assert_allclose(psi, np.array([1, -1, 1, -1]) / 2, atol=1e-15)


def test_phase_vs_expm_diag():
    """exp(-i gamma diag(q)) via scipy expm (Eq. 3)."""
    rng = np.random.default_rng(3)
    N = 32
    q = rng.standard_normal(N)
    psi = _rand_state(N, rng)
    ref = expm(-1j * 0.77 * np.diag(q)) @ psi
    O.phase(psi, q, 0.77)
    np.testing.assert_allclose(psi, ref, atol=1e-14)


def test_expectation_spec_examples():
    """P15: SPEC.md:65-66: uniform over N=4, q=(0,1,2,3) -> 1.5; basis |k> -> q_k."""
    q = np.array([0.0, 1, 2, 3])
    assert O.expectation(O.init_uniform(4), q) == pytest.approx(1.5, abs=1e-15)
    for k in range(4):
        e = np.zeros(4, np.complex128)
        e[k] = 1j
        assert O.expectation(e, q) == q[k]
    assert O.norm2(O.init_uniform(1024)) == pytest.approx(1.0, abs=1e-15)


def test_probabilities():
    rng = np.random.default_rng(5)
    psi = _rand_state(64, rng)
    np.testing.assert_allclose(O.probabilities(psi), np.abs(psi) ** 2, rtol=1e-15)


# ---------------------------------------------------------------- X mixer (P1..P4) ----
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_P1_mixer_x_vs_dense_expm(n):
    """P1: U_M(beta) = expm(-i beta sum_j X_j) (R1) via scipy."""
    rng = np.random.default_rng(100 + n)
    psi = _rand_state(1 << n, rng)
    beta = 0.91
    ref = expm(-1j * beta * O.dense_sum_x(n)) @ psi
    O.mixer_x(psi, beta)
    np.testing.assert_allclose(psi, ref, atol=1e-13)


def test_P1_full_qaoa_vs_dense():
    """P1: full p-layer QAOA vs products of dense expm, n=6, p=3."""
    rng = np.random.default_rng(7)
    n = 6
    u, v = random_regular_graph(n, 3, rng)
    q = O.maxcut_q(n, u, v)
    theta = rng.uniform(0, math.pi, 6)
    W = O.dense_sum_x(n)
    ref = np.full(1 << n, 1 / math.sqrt(1 << n), np.complex128)
    for k in range(3):
        ref = expm(-1j * theta[2 * k] * np.diag(q)) @ ref
        ref = expm(-1j * theta[2 * k + 1] * W) @ ref
    psi = O.evolve_x(n, q, theta)
    np.testing.assert_allclose(psi, ref, atol=1e-12)


def test_P2_basis_state_closed_form():
    """P2: <y|U_M|x0> = cos^{n-d} beta (-i sin beta)^d, d = popcount(x0 ^ y)."""
    n, beta, x0 = 12, 0.6, 0b101100111010
    psi = np.zeros(1 << n, np.complex128)
    psi[x0] = 1.0
    O.mixer_x(psi, beta)
    ys = np.arange(1 << n)
    d = np.array([bin(int(y) ^ x0).count("1") for y in ys])
    ref = np.cos(beta) ** (n - d) * (-1j * np.sin(beta)) ** d
    np.testing.assert_allclose(psi, ref, atol=1e-15)


def test_P3_special_angles():
    """P3: beta=pi/2 -> (-i)^n psi[x ^ (2^n-1)]; beta=pi -> (-1)^n psi; beta=0 -> identity."""
    n = 9
    rng = np.random.default_rng(9)
    psi = _rand_state(1 << n, rng)
    a = psi.copy()
    O.mixer_x(a, math.pi / 2)
    np.testing.assert_allclose(a, (-1j) ** n * psi[np.arange(1 << n) ^ ((1 << n) - 1)], atol=1e-14)
    b = psi.copy()
    O.mixer_x(b, math.pi)
    np.testing.assert_allclose(b, (-1) ** n * psi, atol=1e-14)
    c = psi.copy()
    O.mixer_x(c, 0.0)
    np.testing.assert_array_equal(c, psi)


def test_P4_plus_eigenstate_and_semigroup():
    """P4: U_M(beta)|+> = e^{-i beta n}|+>;  U_M(b1) U_M(b2) = U_M(b1 + b2)."""
    n = 10
    psi = O.init_uniform(1 << n)
    O.mixer_x(psi, 0.37)
    np.testing.assert_allclose(psi, np.exp(-1j * 0.37 * n) / math.sqrt(1 << n), atol=1e-14)
    rng = np.random.default_rng(4)
    s = _rand_state(1 << n, rng)
    a = s.copy()
    O.mixer_x(a, 0.2)
    O.mixer_x(a, 0.5)
    b = s.copy()
    O.mixer_x(b, 0.7)
    np.testing.assert_allclose(a, b, atol=1e-14)


# ---------------------------------------------------------------- invariants (P5, P6) ----
def test_P5_norm_and_P6_theta_zero():
    """P5: |norm^2 - 1| <= 1e-12; P6: theta=0 -> <Q> = mean(q) = -sum(w)/2."""
    wl = make_config("cfg1")
    q = O.maxcut_q(wl.n_qubits, wl.edges_u, wl.edges_v)
    psi = O.evolve_x(wl.n_qubits, q, wl.theta)
    assert abs(O.norm2(psi) - 1) <= 1e-12
    psi0 = O.evolve_x(wl.n_qubits, q, np.zeros(2 * wl.p))
    assert O.expectation(psi0, q) == pytest.approx(-len(wl.edges_u) / 2, rel=1e-13)
    assert len(wl.edges_u) == 15  # 3-regular on 10 vertices -> -7.5


# ---------------------------------------------------------------- analytic p=1 (P7, P8) ----
@pytest.mark.parametrize("n", [4, 5, 8, 11])
def test_P7_ring_closed_form(n):
    """P7: ring C_n, unit weights, q=-cut, p=1:  <Q> = -n/2 + (n/4) sin(4b) sin(2g)."""
    u = np.arange(n)
    v = (u + 1) % n
    uu, vv = np.minimum(u, v), np.maximum(u, v)
    q = O.maxcut_q(n, uu, vv)
    for g, b in [(0.7, 0.3), (2.1, 1.3), (0.05, 2.9)]:
        f = O.expectation(O.evolve_x(n, q, [g, b]), q)
        assert f == pytest.approx(-n / 2 + (n / 4) * math.sin(4 * b) * math.sin(2 * g), abs=1e-12)


def _p1_weighted_closed_form(n, u, v, w, g, b, gw=None):
    """P8: weighted p=1 max-cut closed form (Heisenberg picture), q = -cut_w.  gw: per-edge
    phase angles gamma_e * w_e (ex-QAOA, P18); default g * w."""
    if gw is None:
        gw = [g * x for x in w]
    W = {}
    for a, c, x in zip(u, v, gw):
        W[(int(a), int(c))] = x
        W[(int(c), int(a))] = x
    nbr = {i: set() for i in range(n)}
    for a, c in zip(u, v):
        nbr[int(a)].add(int(c))
        nbr[int(c)].add(int(a))
    total = 0.0
    for a, c, wuv in zip(u, v, w):
        a, c = int(a), int(c)
        Pu = np.prod([math.cos(W[(a, k)]) for k in nbr[a] - {c}])
        Pv = np.prod([math.cos(W[(c, k)]) for k in nbr[c] - {a}])
        T = (nbr[a] & nbr[c])
        U = nbr[a] - T - {c}
        V = nbr[c] - T - {a}
        t1 = 0.5 * math.sin(4 * b) * math.sin(W[(a, c)]) * (Pu + Pv)
        pu = np.prod([math.cos(W[(a, k)]) for k in U])
        pv = np.prod([math.cos(W[(c, k)]) for k in V])
        tm = np.prod([math.cos(W[(a, k)] - W[(c, k)]) for k in T])
        tp = np.prod([math.cos(W[(a, k)] + W[(c, k)]) for k in T])
        t2 = 0.5 * math.sin(2 * b) ** 2 * pu * pv * (tm - tp)
        zz = t1 + t2
        total += wuv / 2 * (zz - 1)
    return total


def test_P8_weighted_p1_closed_form():
    """P8 on G(9, 0.5) with triangles and random weights."""
    rng = np.random.default_rng(8)
    n = 9
    u, v = erdos_renyi_graph(n, 0.5, rng)
    w = rng.uniform(0, 1, len(u))
    q = O.maxcut_q(n, u, v, w)
    for g, b in [(0.9, 0.4), (2.5, 2.2)]:
        f = O.expectation(O.evolve_x(n, q, [g, b]), q)
        assert f == pytest.approx(_p1_weighted_closed_form(n, u, v, w, g, b), abs=1e-12)


# ---------------------------------------------------------------- light cone (P9) ----
@pytest.mark.parametrize("n,d,p,weighted", [(12, 3, 2, False), (14, 3, 2, True), (12, 4, 1, True), (10, 3, 3, False)])
def test_P9_lightcone_equals_full_state(n, d, p, weighted):
    """P9: light-cone <Q> equals the full-state oracle (exact reduction)."""
    rng = np.random.default_rng(n * 10 + p)
    u, v = random_regular_graph(n, d, rng)
    w = rng.uniform(0, 1, len(u)) if weighted else None
    theta = rng.uniform(0, math.pi, 2 * p)
    q = O.maxcut_q(n, u, v, w)
    full = O.expectation(O.evolve_x(n, q, theta), q)
    lc, sizes = O.lightcone_maxcut(n, u, v, w, theta)
    assert lc == pytest.approx(full, rel=1e-12, abs=1e-12)
    assert sizes.max() <= n


# ---------------------------------------------------------------- circulant (P10, P11) ----
@pytest.mark.parametrize("N", [2, 7, 13, 16, 31, 60])
def test_P11_circulant_dense_vs_expm_symmetric_row(N):
    """P11: symmetric first row w: C = circulant(w), lambda = fft(w) (R4) -> expm(-i b C) psi."""
    rng = np.random.default_rng(N)
    w = rng.uniform(-1, 1, N)
    w = 0.5 * (w + np.roll(w[::-1], 1))  # w_k = w_{N-k}
    C = circulant(w)
    assert np.allclose(C, C.T)
    lam = np.fft.fft(w).real
    psi = _rand_state(N, rng)
    ref = expm(-1j * 0.83 * C) @ psi
    O.mixer_circulant_dense(psi, lam, 0.83)
    np.testing.assert_allclose(psi, ref, atol=1e-12)


@pytest.mark.parametrize("N", [5, 64, 97, 210, 1024])
def test_P11_circulant_dense_vs_numpy_fft(N):
    """P11: arbitrary real spectrum: ifft(exp(-i b lambda) * fft(psi)) (numpy pocketfft)."""
    rng = np.random.default_rng(N + 1)
    lam = rng.standard_normal(N) * 3
    psi = _rand_state(N, rng)
    ref = np.fft.ifft(np.exp(-1j * 1.9 * lam) * np.fft.fft(psi))
    O.mixer_circulant_dense(psi, lam, 1.9)
    np.testing.assert_allclose(psi, ref, atol=1e-12)


@pytest.mark.parametrize("N", [2, 6, 24, 120])
def test_P10_complete_closed_form_vs_expm_laplacian(N):
    """P10: K_N Laplacian L = N I - J has spectrum (0, N, ..., N) (cfg3, R5).
    Closed form vs expm(-i b L) and vs the dense circulant definition."""
    rng = np.random.default_rng(N)
    psi = _rand_state(N, rng)
    L = N * np.eye(N) - np.ones((N, N))
    ref = expm(-1j * 0.41 * L) @ psi
    a = psi.copy()
    O.mixer_complete(a, 0.41, 0.0, float(N))
    np.testing.assert_allclose(a, ref, atol=1e-12)
    b = psi.copy()
    lam = np.full(N, float(N))
    lam[0] = 0.0
    O.mixer_circulant_dense(b, lam, 0.41)
    np.testing.assert_allclose(b, ref, atol=1e-12)
    # adjacency of K_N: spectrum (N-1, -1, ..., -1)
    A = np.ones((N, N)) - np.eye(N)
    c = psi.copy()
    O.mixer_complete(c, 0.41, N - 1.0, -1.0)
    np.testing.assert_allclose(c, expm(-1j * 0.41 * A) @ psi, atol=1e-12)


def test_P10_complete_at_cfg3_size_vs_numpy_fft():
    """P10 at N = 10! (cfg3 size): closed form vs numpy.fft definition."""
    N = math.factorial(10)
    rng = np.random.default_rng(33)
    psi = _rand_state(N, rng)
    lam = np.full(N, float(N))
    lam[0] = 0.0
    ref = np.fft.ifft(np.exp(-1j * 1.1 * lam) * np.fft.fft(psi))
    O.mixer_complete(psi, 1.1, 0.0, float(N))
    np.testing.assert_allclose(psi, ref, atol=1e-12)


def test_P4_circulant_uniform_and_semigroup():
    """P4 for the circulant: uniform state is the j=0 mode -> e^{-i b lambda_0} uniform;
    semigroup U(b1)U(b2) = U(b1+b2)."""
    N = 48
    rng = np.random.default_rng(2)
    lam = rng.standard_normal(N)
    u = O.init_uniform(N)
    O.mixer_circulant_dense(u, lam, 0.7)
    np.testing.assert_allclose(u, np.exp(-1j * 0.7 * lam[0]) / math.sqrt(N), atol=1e-14)
    s = _rand_state(N, rng)
    a = s.copy()
    O.mixer_circulant_dense(a, lam, 0.3)
    O.mixer_circulant_dense(a, lam, 0.9)
    b = s.copy()
    O.mixer_circulant_dense(b, lam, 1.2)
    np.testing.assert_allclose(a, b, atol=1e-12)


def test_qwoa_evolve_complete_vs_dense():
    """Full QWOA evolution closed-form mixer vs dense circulant definition."""
    N = 120
    rng = np.random.default_rng(12)
    q = rng.standard_normal(N)
    theta = rng.uniform(0, math.pi, 8)
    lam = np.full(N, float(N))
    lam[0] = 0.0
    a = O.evolve_complete(q, theta, 0.0, float(N))
    b = O.evolve_circulant_dense(q, lam, theta)
    np.testing.assert_allclose(a, b, atol=1e-12)
    assert abs(O.norm2(a) - 1) < 1e-12


# ---------------------------------------------------------------- sparse (P12) ----
def test_P12_sparse_dense_spec_example():
    """P12: SPEC.md:159-161: N=2, W=X, t=pi/2, |0> -> -i|1>."""
    out = O.mixer_sparse_dense(np.array([1.0, 0.0], np.complex128), O.dense_sum_x(1), math.pi / 2)
    np.testing.assert_allclose(out, [0, -1j], atol=1e-15)


# ---------------------------------------------------------------- FD gradient (P13) ----
def test_P13_central_difference_gradient_vs_analytic_ring():
    """P13: batch order [theta, theta+h e1, theta-h e1, ...] (R12) and central differences
    reproduce d<Q>/d(gamma, beta) of the P7 closed form to O(h^2) + roundoff."""
    n = 8
    u = np.arange(n)
    v = (u + 1) % n
    q = O.maxcut_q(n, np.minimum(u, v), np.maximum(u, v))
    theta = np.array([0.7, 0.3])
    h = 1e-6
    B = fd_batch_thetas(theta, h)
    f = np.array([O.expectation(O.evolve_x(n, q, t), q) for t in B])
    grad = [(f[1 + 2 * k] - f[2 + 2 * k]) / (2 * h) for k in range(2)]
    g, b = theta
    dg = (n / 4) * math.sin(4 * b) * 2 * math.cos(2 * g)
    db = (n / 4) * 4 * math.cos(4 * b) * math.sin(2 * g)
    assert grad[0] == pytest.approx(dg, abs=2e-8)
    assert grad[1] == pytest.approx(db, abs=2e-8)


# ---------------------------------------------------------------- inputs module ----
def test_input_recipes():
    for name, (N, p) in {"cfg1": (1024, 2), "cfg4": (1 << 30, 3), "cfg5": (1 << 34, 2)}.items():
        wl = make_config(name)
        assert wl.dim == N and wl.p == p and len(wl.theta) == 2 * p
        assert np.all((wl.theta > 0) & (wl.theta < math.pi))
        deg = np.bincount(np.concatenate([wl.edges_u, wl.edges_v]), minlength=wl.n_qubits)
        assert len(set(deg.tolist())) == 1
        assert np.all(wl.edges_u < wl.edges_v)
    wl2 = make_config("cfg2")
    assert wl2.batch_thetas.shape == (21, 10)
    wl3 = make_config("cfg3", n_override=720)
    assert wl3.dim == 720 and wl3.q.shape == (720,)
    # determinism
    assert np.array_equal(make_config("cfg4").edges_u, make_config("cfg4").edges_u)


# ---------------------------------------------------------------- P16 QAOAz parity mixer ----
_PX = np.array([[0, 1], [1, 0]], complex)
_PY = np.array([[0, -1j], [1j, 0]], complex)


def _dense_pauli(n, ops):
    """Dense operator of a Pauli product {qubit: 2x2}; qubit j <-> bit j of the index (R8), so
    qubit n-1 is the leftmost Kronecker factor."""
    M = np.array([[1.0 + 0j]])
    for j in reversed(range(n)):
        M = np.kron(M, ops.get(j, np.eye(2)))
    return M


def _dense_B(n, pairs):
    B = np.zeros((1 << n, 1 << n), complex)
    for a, b in pairs:
        B += _dense_pauli(n, {a: _PX, b: _PX}) + _dense_pauli(n, {a: _PY, b: _PY})
    return B


def test_P16_dense_xy_term_spec_example():
    """on 2 qubits B_odd = X0X1 + Y0Y1 maps |01> to 2|10> (and kills |00>, |11>)."""
    B = _dense_B(2, [(0, 1)])
    e = np.eye(4)
    # index x = bit0 + 2 bit1: |q1 q0> = |01> is x = 1, |10> is x = 2
    assert np.allclose(B @ e[1], 2 * e[2]) and np.allclose(B @ e[2], 2 * e[1])
    assert np.allclose(B @ e[0], 0) and np.allclose(B @ e[3], 0)


@pytest.mark.parametrize("n,seq", [(2, [0, 1]), (3, [0, 1, 2]), (4, [3, 1, 0, 2]), (5, [0, 1, 2, 3, 4]),
                                   (6, [5, 2, 4]), (7, [6, 0, 3, 1, 5, 2, 4])])
def test_P16_parity_mixer_vs_dense_expm(n, seq):
    """U_parity(t) = e^{-itB_last} e^{-itB_even} e^{-itB_odd} (PAPER.md Eq. qaoaz_mixers) built from
    dense Pauli matrices and scipy expm, against the oracle's pair rotations."""
    rng = np.random.default_rng(n + len(seq))
    t = float(rng.uniform(0, math.pi))
    odd, even, last = O.parity_pairs(seq)
    U = expm(-1j * t * _dense_B(n, last)) @ expm(-1j * t * _dense_B(n, even)) @ expm(-1j * t * _dense_B(n, odd))
    psi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    got = O.mixer_parity(psi.copy(), seq, t)
    assert np.max(np.abs(got - U @ psi)) < 1e-12


def test_P16_parity_conservation_and_special_angle():
    """Hamming weight on the subsequence is conserved (|0011> stays in weight 2); at
    t = pi/2 every pair rotation is Z_a Z_b, so U = prod over all pairs of (-1)^(x_a xor x_b)."""
    n, seq = 6, [0, 1, 2, 3, 4, 5]
    psi = np.zeros(1 << n, complex)
    psi[0b000011] = 1.0
    out = O.mixer_parity(psi.copy(), seq, 0.73)
    w = np.array([bin(x).count("1") for x in range(1 << n)])
    assert np.sum(np.abs(out[w != 2]) ** 2) < 1e-12 and abs(np.linalg.norm(out) - 1) < 1e-12
    rng = np.random.default_rng(3)
    seq = [4, 0, 2, 5, 1]
    phi = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    odd, even, last = O.parity_pairs(seq)
    sign = np.ones(1 << n)
    for a, b in odd + even + last:
        sign *= np.array([(-1.0) ** (((x >> a) ^ (x >> b)) & 1) for x in range(1 << n)])
    assert np.max(np.abs(O.mixer_parity(phi.copy(), seq, math.pi / 2) - sign * phi)) < 1e-12


# ---------------------------------------------------------------- permutation subspaces (P17) ----
@pytest.mark.parametrize("m,k", [(1, 1), (3, 3), (4, 2), (5, 5), (6, 3), (7, 7), (8, 1)])
def test_P17_kperm_unrank_is_itertools_order(m, k):
    """P17: rank r <-> the r-th k-permutation in lexicographic order (R23): kperm_unrank against
    itertools.permutations (library order), over every rank; the count is m!/(m-k)!."""
    import itertools
    ref = list(itertools.permutations(range(m), k))
    assert O.kperm_count(m, k) == len(ref)
    for r, pi in enumerate(ref):
        assert tuple(O.kperm_unrank(m, k, r)) == pi


def test_P17_kperm_lehmer_code_definition():
    """P17: the Lehmer code d_a = #{unused elements < s_a} read as a mixed-radix number with
    radices (m-a)... gives back the rank (Knuth's definition of the factorial number system)."""
    m, k = 9, 5
    for r in [0, 1, 2, 1000, 7777, O.kperm_count(m, k) - 1]:
        pi = O.kperm_unrank(m, k, r)
        rank = 0
        for a in range(k):
            d = sum(1 for x in pi[a + 1:] if x < pi[a]) + sum(
                1 for x in range(m) if x not in pi and x < pi[a])
            rank = rank * (m - a) + d
        assert rank == r


def test_P17_tsp_worked_example():
    """P17 worked example, by hand: m = k = 3, directed 3-cycle F (F[a][(a+1)%3] = 1),
    D = [[0,1,2],[4,0,8],[16,32,0]] (asymmetric).  Lexicographic tours and their costs:
    012: D01+D12+D20 = 1+8+16 = 25; 021: D02+D21+D10 = 2+32+4 = 38; 102: D10+D02+D21 = 38;
    120: D12+D20+D01 = 25; 201: D20+D01+D12 = 25; 210: D21+D10+D02 = 38."""
    F = [[0, 1, 0], [0, 0, 1], [1, 0, 0]]
    D = [[0, 1, 2], [4, 0, 8], [16, 32, 0]]
    assert list(O.kperm_qualities(3, 3, F, D)) == [25.0, 38.0, 38.0, 25.0, 25.0, 38.0]
    # a linear (assignment) term: C[a][s_a]
    C = [[100, 200, 300], [0, 0, 0], [0, 0, 7]]
    assert list(O.kperm_qualities(3, 3, F, D, C)) == [25 + 100 + 7, 38 + 100, 38 + 200 + 7,
                                                      25 + 200, 25 + 300, 38 + 300]


@pytest.mark.parametrize("m,k", [(6, 6), (7, 4), (5, 2)])
def test_P17_kperm_sum_closed_form(m, k):
    """P17: sum over all k-permutations of sum_ab F_ab D_{s_a s_b} + C_{a s_a} equals
    sum_{a!=b} F_ab * sum_{i!=j} D_ij * (m-2)!/(m-k)! + sum_a F_aa * tr D * (m-1)!/(m-k)!
    + sum_a sum_i C_ai * (m-1)!/(m-k)! (each ordered pair / element is equally often used)."""
    rng = np.random.default_rng(m * 10 + k)
    F = rng.uniform(-1, 1, (k, k))
    D = rng.uniform(-1, 1, (m, m))
    C = rng.uniform(-1, 1, (k, m))
    q = O.kperm_qualities(m, k, F, D, C)
    off = F.sum() - np.trace(F)
    ref = off * (D.sum() - np.trace(D)) * (math.perm(m - 2, k - 2) if k >= 2 else 0)
    ref += np.trace(F) * np.trace(D) * math.perm(m - 1, k - 1)
    ref += C.sum() * math.perm(m - 1, k - 1)
    assert q.sum() == pytest.approx(ref, rel=1e-12, abs=1e-9)


def test_P17_tsp_rotation_invariance():
    """P17: a closed tour's cost does not depend on its starting city: with F the directed
    m-cycle, q(s) = q(rotate(s)) for every s (catches a transposed F or D index)."""
    m = 6
    rng = np.random.default_rng(17)
    D = rng.uniform(0, 1, (m, m))
    F = np.zeros((m, m))
    for a in range(m):
        F[a, (a + 1) % m] = 1
    import itertools
    perms = list(itertools.permutations(range(m)))
    q = O.kperm_qualities(m, m, F, D)
    index = {p: i for i, p in enumerate(perms)}
    for i, pi in enumerate(perms):
        rot = pi[1:] + pi[:1]
        assert q[index[rot]] == pytest.approx(q[i], abs=1e-14)
        rev = tuple(reversed(pi))  # the reversed tour costs sum D^T: differs for asymmetric D
        assert abs(q[index[rev]] - sum(D[pi[(a + 1) % m], pi[a]] for a in range(m))) < 1e-12


# ---------------------------------------------------------------- ex-QAOA (P18) ----
def test_P18_ex_qaoa_equal_gammas_is_qaoa():
    """P18: with gamma_{i,e} = gamma_i for every term, Eq. phase_shift_qaoa_ex is exp(-i gamma_i Q)
    (R25: the terms sum to q), so ex-QAOA reduces to QAOA (Eq. qaoa) amplitude by amplitude."""
    rng = np.random.default_rng(18)
    n = 8
    u, v = erdos_renyi_graph(n, 0.5, rng)
    w = rng.uniform(0, 1, len(u))
    m = len(u)
    theta = rng.uniform(0, math.pi, 4)
    tex = np.concatenate([np.r_[np.full(m, theta[2 * i]), theta[2 * i + 1]] for i in range(2)])
    a = O.evolve_ex(n, u, v, w, tex)
    b = O.evolve_x(n, O.maxcut_q(n, u, v, w), theta)
    assert np.max(np.abs(a - b)) < 1e-13


def test_P18_ex_qaoa_vs_dense_pauli_expm():
    """P18: ex-QAOA against dense matrices built from Pauli Z / X Kronecker products:
    Sigma_e = -w_e (I - Z_u Z_v) / 2, layer = expm(-i t sum_j X_j) expm(-i sum_e gamma_e Sigma_e)."""
    rng = np.random.default_rng(181)
    n = 5
    u, v = erdos_renyi_graph(n, 0.7, rng)
    w = rng.uniform(0.2, 1, len(u))
    m = len(u)
    I2, Z = np.eye(2), np.diag([1.0, -1.0])

    def op(j, P):  # qubit j = bit j of the index (R8): kron order puts qubit n-1 first
        out = np.array([[1.0]])
        for b in reversed(range(n)):
            out = np.kron(out, P if b == j else I2)
        return out

    Sig = [-w[e] * (np.eye(1 << n) - op(u[e], Z) @ op(v[e], Z)) / 2 for e in range(m)]
    Xs = O.dense_sum_x(n)
    theta = rng.uniform(0, math.pi, 2 * (m + 1))
    psi = np.full(1 << n, (1 << n) ** -0.5, np.complex128)
    for i in range(2):
        th = theta[i * (m + 1):(i + 1) * (m + 1)]
        H = sum(th[e] * Sig[e] for e in range(m))
        psi = expm(-1j * Xs * th[m]) @ (expm(-1j * H) @ psi)
    assert np.max(np.abs(O.evolve_ex(n, u, v, w, theta) - psi)) < 1e-12


def test_P18_ex_qaoa_p1_closed_form():
    """P18: at p = 1 the P8 closed form holds with the per-edge phase angles gamma_e w_e in place
    of gamma w (the Heisenberg-picture derivation only uses the products); <Q> keeps w."""
    rng = np.random.default_rng(182)
    n = 9
    u, v = erdos_renyi_graph(n, 0.5, rng)
    w = rng.uniform(0, 1, len(u))
    m = len(u)
    q = O.maxcut_q(n, u, v, w)
    for _ in range(2):
        th = rng.uniform(0, math.pi, m + 1)
        f = O.expectation(O.evolve_ex(n, u, v, w, th), q)
        ref = _p1_weighted_closed_form(n, u, v, w, 0.0, th[m], gw=list(th[:m] * w))
        assert f == pytest.approx(ref, abs=1e-12)


# ---------------------------------------------------------------- evolution loops (P19) ----
# The p-layer products of the QWOA, QAOAz and generic-sparse oracles, each pinned against a
# product of dense unitaries built by a route the oracle does not use (closed-form matrices,
# Pauli Kronecker products, numpy.linalg.eigh).  PAPER.md:46-51 (Eq. 1): layer k applies
# U_Q(gamma_k) then U_M(beta_k); layer 1 acts first (R6); theta = [g1, b1, ...] (R7).
# Each test also checks that the plausible mistakes -- mixer before phase, gamma/beta swapped,
# layers in reverse order -- would NOT pass, so the pin is sensitive to the loop structure.

def _dense_product(psi0, q, mixer_u, theta, order="pm", swap=False, reverse=False):
    """Dense reference: for k = 1..p, psi <- U_M(b_k) U_Q(g_k) psi with U_Q = expm(-i g diag q)
    written as the diagonal exp(-i g q_x) (Eq. 3) and U_M = mixer_u(b)."""
    psi = np.array(psi0, np.complex128)
    p = len(theta) // 2
    layers = list(range(p))[::-1] if reverse else range(p)
    for k in layers:
        g, b = theta[2 * k], theta[2 * k + 1]
        if swap:
            g, b = b, g
        UQ = np.exp(-1j * g * np.asarray(q))
        if order == "pm":
            psi = mixer_u(b) @ (UQ * psi)
        else:
            psi = UQ * (mixer_u(b) @ psi)
    return psi


def _assert_loop_pinned(got, psi0, q, mixer_u, theta, tol=1e-12):
    ref = _dense_product(psi0, q, mixer_u, theta)
    assert np.max(np.abs(got - ref)) < tol
    for kw in ({"order": "mp"}, {"swap": True}, {"reverse": True}):
        bad = _dense_product(psi0, q, mixer_u, theta, **kw)
        assert np.max(np.abs(bad - ref)) > 1e-4, kw  # the pin distinguishes this mistake


def _expm_hermitian(H, t):
    """exp(-i t H) for a real symmetric / Hermitian H by numpy.linalg.eigh (not scipy expm)."""
    lam, V = np.linalg.eigh(H)
    return (V * np.exp(-1j * t * lam)) @ V.conj().T


@pytest.mark.parametrize("N,lam0,lam_rest", [(24, 0.0, 24.0), (120, 0.0, 120.0), (37, 1.5, -0.4)])
def test_P19_qwoa_evolve_complete_vs_dense_product(N, lam0, lam_rest):
    """QWOA (PAPER.md:298 Eq. qwoa) with the complete-graph-family spectrum: the circulant with
    lambda = (lam0, c, ..., c) is the matrix c I + (lam0 - c)/N J (J = all ones: the j = 0 mode is
    the uniform vector).  cfg3's Laplacian (R5) is lam0 = 0, c = N, i.e. N I - J."""
    rng = np.random.default_rng(N)
    q = rng.standard_normal(N)
    theta = rng.uniform(0, math.pi, 8)
    C = lam_rest * np.eye(N) + (lam0 - lam_rest) / N * np.ones((N, N))
    psi0 = np.full(N, 1 / math.sqrt(N), np.complex128)
    psi0 = psi0 * np.exp(1j * rng.uniform(0, 2 * math.pi, N))  # a non-uniform start exercises the mixer
    got = O.evolve_complete(q, theta, lam0, lam_rest, psi0=psi0)
    _assert_loop_pinned(got, psi0, q, lambda b: _expm_hermitian(C, b), theta)
    # default psi0 = |+> (a1)
    got = O.evolve_complete(q, theta, lam0, lam_rest)
    ref = _dense_product(np.full(N, 1 / math.sqrt(N), np.complex128), q, lambda b: _expm_hermitian(C, b), theta)
    assert np.max(np.abs(got - ref)) < 1e-12


@pytest.mark.parametrize("N", [16, 45, 64])
def test_P19_qwoa_evolve_circulant_dense_vs_dense_product(N):
    """QWOA with an arbitrary symmetric circulant mixer: the dense matrix is
    scipy's circulant(c) of a random symmetric first column c (c_k = c_{N-k}); its spectrum by
    forward-DFT bin is lambda_j = sum_k c_k cos(2 pi j k / N), written out here (R4)."""
    rng = np.random.default_rng(500 + N)
    c = rng.standard_normal(N)
    c = 0.5 * (c + np.roll(c[::-1], 1))
    k = np.arange(N)
    lam = np.array([np.sum(c * np.cos(2 * math.pi * ((j * k) % N) / N)) for j in range(N)])
    C = circulant(c)
    assert np.allclose(C, C.T)
    q = rng.standard_normal(N)
    theta = rng.uniform(0, math.pi, 6)
    psi0 = _rand_state(N, rng)
    got = O.evolve_circulant_dense(q, lam, theta, psi0=psi0)
    _assert_loop_pinned(got, psi0, q, lambda b: _expm_hermitian(C, b), theta)


@pytest.mark.parametrize("n,seq", [(3, [0, 1, 2]), (5, [4, 0, 2, 1, 3]), (6, [1, 3, 5, 0]), (7, [6, 0, 3, 1, 5, 2, 4])])
def test_P19_qaoaz_evolve_parity_vs_dense_product(n, seq):
    """QAOAz (PAPER.md:213-248 Eqs. parity_terms / qaoaz_mixers / qaoaz): per layer the phase, then
    e^{-itB_odd}, e^{-itB_even}, e^{-itB_last} with each B a sum of dense X_aX_b + Y_aY_b Pauli
    Kronecker products (R19), exponentiated by eigh."""
    rng = np.random.default_rng(n * 10 + len(seq))
    odd, even, last = O.parity_pairs(seq)
    Bs = [_dense_B(n, pr) for pr in (odd, even, last)]

    def U(t):
        M = np.eye(1 << n, dtype=complex)
        for B in Bs:
            M = _expm_hermitian(B, t) @ M
        return M
    q = rng.standard_normal(1 << n)
    theta = rng.uniform(0, math.pi, 6)
    psi0 = _rand_state(1 << n, rng)
    got = O.evolve_parity(n, q, seq, theta, psi0)
    _assert_loop_pinned(got, psi0, q, U, theta)


@pytest.mark.parametrize("N,density", [(12, 0.3), (64, 0.08)])
def test_P19_generic_sparse_evolve_vs_dense_product(N, density):
    """Generic QVA with a sparse symmetric mixer W (PAPER.md:46-51 Eq. 1, :72-77 Eq. 4, :333): the
    oracle's evolve_sparse_dense (scipy expm per layer) against exp(-i beta W) by eigh."""
    rng = np.random.default_rng(N)
    W = np.where(rng.uniform(size=(N, N)) < density, rng.uniform(-1, 1, (N, N)), 0.0)
    W = np.triu(W, 1)
    W = W + W.T + np.diag(rng.uniform(-0.5, 0.5, N) * (rng.uniform(size=N) < 0.5))
    q = rng.standard_normal(N)
    theta = rng.uniform(0, math.pi, 8)
    psi0 = _rand_state(N, rng)
    got = O.evolve_sparse_dense(q, W, theta, psi0=psi0)
    _assert_loop_pinned(got, psi0, q, lambda b: _expm_hermitian(W, b), theta)
    got = O.evolve_sparse_dense(q, W, theta)
    ref = _dense_product(np.full(N, 1 / math.sqrt(N), np.complex128), q, lambda b: _expm_hermitian(W, b), theta)
    assert np.max(np.abs(got - ref)) < 1e-12


# ---------------------------------------------------------------- P20: FFT-route QWOA oracle ----
@pytest.mark.parametrize("N", [12, 97, 720, 1001])
def test_P20_evolve_circulant_fft_vs_dense(N):
    """P20: the numpy-FFT QWOA evolution (large-N oracle of the circulant mixer)
    equals the O(N^2) dense-definition evolution (itself pinned by P11 / P19) for a random real
    spectrum and a random initial state; a swapped gamma/beta fails."""
    rng = np.random.default_rng(900 + N)
    q = rng.standard_normal(N)
    lam = rng.standard_normal(N) * 3
    theta = rng.uniform(0, math.pi, 6)
    psi0 = _rand_state(N, rng)
    ref = O.evolve_circulant_dense(q, lam, theta, psi0)
    got = O.evolve_circulant_fft(q, lam, theta, psi0)
    np.testing.assert_allclose(got, ref, atol=1e-11)
    swapped = O.evolve_circulant_fft(q, lam, theta.reshape(-1, 2)[:, ::-1].ravel(), psi0)
    assert np.max(np.abs(swapped - ref)) > 1e-3
