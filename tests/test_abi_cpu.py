"""C-ABI library checks that need no GPU (`-m "not gpu"`): the library loads, exports every
symbol include/qva.h declares, and its host-only logic (partition, batch split, X-mixer pass
schedule) is right."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "qva.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qva_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def Q():
    import paper_2110_03963_b200 as Q
    return Q


def test_library_exports_every_declared_symbol(Q):
    import ctypes
    lib = ctypes.CDLL(Q.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert "sm_100a" in Q.qva_version()


def test_library_is_sm100a_only(Q):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", Q.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


@pytest.mark.parametrize("N,world,sizes,offsets", [
    (16, 4, [4, 4, 4, 4], [0, 4, 8, 12]),
    (10, 4, [3, 3, 2, 2], [0, 3, 6, 8]),       # SPEC.md:46 remainder to leading ranks (R16)
    (2, 4, [1, 1, 0, 0], [0, 1, 2, 2]),        # SPEC.md:47 zero-size ranks
    (1 << 34, 8, [1 << 31] * 8, [r << 31 for r in range(8)]),
])
def test_partition(Q, N, world, sizes, offsets):
    """Eqs. local_i / offset."""
    got = [Q.qva_partition(N, world, r) for r in range(world)]
    assert [g[0] for g in got] == sizes
    assert [g[1] for g in got] == offsets


def test_partition_errors(Q):
    with pytest.raises(Q.QvaError):
        Q.qva_partition(16, 0, 0)
    with pytest.raises(Q.QvaError):
        Q.qva_partition(16, 2, 2)


@pytest.mark.parametrize("B,world", [(21, 1), (21, 2), (21, 8), (3, 8), (0, 4)])
def test_batch_partition(Q, B, world):
    parts = [Q.qva_batch_partition(B, world, r) for r in range(world)]
    covered = []
    for f, c in parts:
        covered += list(range(f, f + c))
    assert covered == list(range(B))
    counts = [c for _, c in parts]
    assert max(counts) - min(counts) <= 1


@pytest.mark.parametrize("n,p", [(12, 1), (13, 2), (20, 5), (21, 3), (24, 2), (30, 3), (31, 2), (33, 4), (34, 2)])
def test_x_schedule_covers_every_rotation_once(Q, n, p):
    """The pass schedule applies each of the n single-qubit rotations exactly once per layer
    and exactly p phases, with one HBM pass per tile set plus shared
    layer-boundary passes."""
    sched = Q.qva_x_schedule(n, p)
    rots = sum(s[1] + s[3] for s in sched)
    phases = sum(s[2] for s in sched)
    assert rots == n * p
    assert phases == p
    n_sets = 1 + -(-(n - 12) // 9) if n > 12 else 1
    # every layer boundary shares a pass: passes = (n_sets - 1) * p + 1 for n_sets >= 2
    if n_sets >= 2:
        assert len(sched) == (n_sets - 1) * p + 1
    assert sched[0][1] == 0 and sched[0][2] == 1  # first pass: phase then rotations


def test_x_schedule_n30_p3(Q):
    """cfg4: 7 passes for 3 layers (vs 9 without layer-boundary fusion)."""
    sched = Q.qva_x_schedule(30, 3)
    assert len(sched) == 7


@pytest.mark.parametrize("n,p", [(21, 1), (21, 4), (22, 2), (24, 3), (29, 2), (30, 1), (30, 3), (31, 2), (34, 3)])
def test_permuted_schedule_order(Q, n, p):
    """Permuted single-shard schedule: in stream order every logical qubit is rotated exactly once
    per layer, layer k's rotations come after phase k and before phase k+1 (Eq. qaoa, PAPER.md:185:
    U_M(beta_k) U_Q(gamma_k), layer 1 first; reading R6), the expectation is fused into the last
    pass only, and every pass fits the 5 TMA dims of one tensor map."""
    sched = Q.qva_x_schedule_permuted(n, p)
    events = []  # ("P", k) / ("R", k, mask) in application order
    for s in sched:
        assert s["dims"] <= 5
        if s["r1"]:
            events.append(("R", s["a1"], s["r1"]))
        if s["phase"] >= 0:
            events.append(("P", s["phase"]))
        if s["r2"]:
            events.append(("R", s["a2"], s["r2"]))
    assert [s["expect"] for s in sched] == [0] * (len(sched) - 1) + [1]
    layer = -1
    done = 0
    for e in events:
        if e[0] == "P":
            assert e[1] == layer + 1 and (layer < 0 or done == (1 << n) - 1)
            layer, done = e[1], 0
        else:
            assert e[1] == layer and not (done & e[2])
            done |= e[2]
    assert layer == p - 1 and done == (1 << n) - 1
    # every pass after the first reads the 64-KiB-stride window at bit 12
    assert sched[0]["window"] == 3 and all(s["window"] == 12 for s in sched[1:])


def test_permuted_schedule_n30_p3(Q):
    """cfg4 keeps 2p+1 = 7 passes in the permuted schedule."""
    assert len(Q.qva_x_schedule_permuted(30, 3)) == 7


def _smooth13(m):
    for p in (2, 3, 5, 7, 11, 13):
        while m % p == 0:
            m //= p
    return m == 1


def test_circulant_plan_shapes(Q):
    """Every N gets an FFT plan (Sec. 3; north_star (c): arbitrary N): 13-smooth
    N <= 4096 run whole in one CTA, N = N1*N2 with 13-smooth factors <= 8192 use the four-step
    mixed-radix form, anything else Bluestein with a 13-smooth length M >= 2N - 1."""
    rng = np.random.default_rng(5)
    Ns = list(range(1, 300)) + [4096, 4097, 4099, 5040, 6144, 8191, 8192, 3628800, 65537, 1000003,
                                362881, 2 ** 22, 3 ** 13, 10 ** 7] + [int(x) for x in rng.integers(300, 4_000_000, 40)]
    for N in Ns:
        sh = Q.qva_circulant_plan_shape(N)
        assert sh["kind"] in (0, 1, 2), (N, sh)
        if sh["kind"] == 0:
            assert N <= 4096 and _smooth13(N) and sh["M"] == N
            continue
        assert sh["M1"] * sh["M2"] == sh["M"] and _smooth13(sh["M1"]) and _smooth13(sh["M2"])
        assert sh["M2"] <= 8192 and sh["cw"] in (1, 2, 4, 8) and sh["M1"] % sh["rb"] == 0
        if sh["kind"] == 1:
            assert sh["M"] == N and _smooth13(N)
        else:
            assert sh["M"] >= 2 * N - 1


@pytest.mark.parametrize("N,G", [(3628800, 2), (3628800, 4), (3628800, 8), (6144, 8), (40320, 4), (1 << 20, 8)])
def test_sharded_circulant_plan_shapes(Q, N, G):
    """Sharded QWOA: the four-step split keeps whole row blocks (G | M1) and
    whole column blocks (G | M2) on every shard; non-smooth N has no sharded plan."""
    sh = Q.qva_circulant_plan_shape(N, G)
    assert sh["kind"] == 1 and sh["M"] == N and sh["M1"] * sh["M2"] == N
    assert sh["M1"] % G == 0 and sh["M2"] % G == 0


@pytest.mark.parametrize("N,G,force", [(479001600, 1, False), (479001600, 8, False), (6227020800, 1, False),
                                       (40320, 1, True), (3628800, 4, True)])
def test_three_level_circulant_plan_shapes(Q, N, G, force):
    """NEXT-4: above 8192^2 states (12! = 4.8e8, 13! = 6.2e9) the circulant mixer uses a three-level
    four-step split N = M1 * Mi1 * Mi2 with 13-smooth factors (column lengths <= 1024, inner row
    <= 8192); sharded plans keep G | M1 and G | Mi1 * Mi2."""
    sh = Q.qva_circulant_plan_shape(N, G, force)
    assert sh["kind"] == 3 and sh["levels"] == 3 and sh["M"] == N
    assert sh["M1"] * sh["Mi1"] * sh["Mi2"] == N and sh["M2"] == sh["Mi1"] * sh["Mi2"]
    assert sh["M1"] <= 1024 and sh["Mi1"] <= 1024 and sh["Mi2"] <= 8192
    assert all(_smooth13(x) for x in (sh["M1"], sh["Mi1"], sh["Mi2"]))
    assert sh["M1"] % G == 0 and sh["M2"] % G == 0


def test_sharded_circulant_prime_unsupported(Q):
    with pytest.raises(Q.QvaError) as ei:
        Q.qva_circulant_plan_shape(1000003, 2)
    assert ei.value.status == 5


def test_plan_create_without_gpu_fails_cleanly(Q):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(1 << 10, "x", n_qubits=10)
    assert ei.value.status in (7, 6)  # QVA_ERR_CUDA / OUT_OF_MEMORY


def test_plan_argument_errors(Q):
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(1000, "x", n_qubits=10)
    assert ei.value.status == 5  # UNSUPPORTED: dim != 2^n
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(1 << 20, "x", n_qubits=20, virtual_shards=3)
    assert ei.value.status == 5  # non power of two shards
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(721, "circulant", world=2, rank=0)  # sharded QWOA needs shards | dim
    assert ei.value.status == 5
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(720, "sparse", virtual_shards=2)  # sparse mixer: row blocks over real ranks only
    assert ei.value.status == 5
    with pytest.raises(Q.QvaError) as ei:
        Q.Plan(1 << 12, "parity", n_qubits=12, world=2, rank=0)  # sharded QAOAz: replicated mode only
    assert ei.value.status == 5


# ---------------------------------------------------------------- QAOAz window schedule (host) ----
@pytest.mark.parametrize("n,seed", [(6, 0), (12, 1), (20, 2), (28, 3), (33, 4), (40, 5)])
def test_parity_window_schedule(Q, n, seed):
    """The parity mixer's window passes (qva_parity_schedule, host-only): every term of B_odd,
    B_even and B_last (reading R19; the oracle's parity_pairs) applied exactly once, inside its
    window (<= 12 bits, bits 0..2 included), after every earlier-group term it shares a qubit with."""
    import oracle as O
    rng = np.random.default_rng(seed)
    for trial in range(4):
        if trial == 0:
            seq = list(range(n))
        else:
            K = int(rng.integers(2, n + 1))
            seq = [int(x) for x in rng.permutation(n)[:K]]
        odd, even, last = O.parity_pairs(seq)
        groups = [(0, t) for t in odd] + [(1, t) for t in even] + [(2, t) for t in last]
        wins = Q.qva_parity_schedule(n, seq)
        order = []
        for bits, pairs in wins:
            assert len(bits) <= 12 and bits == sorted(bits) and len(set(bits)) == len(bits)
            assert all(b in bits for b in range(min(3, n)))
            for a, b in pairs:
                assert a in bits and b in bits
                order.append((a, b))
        assert len(order) == len(groups)
        pos = {}
        for i, (a, b) in enumerate(order):
            pos[frozenset((a, b))] = i
        for g, (a, b) in groups:
            key = frozenset((a, b))
            assert key in pos
            for g2, (c, d) in groups:
                if g2 < g and {c, d} & {a, b}:
                    assert pos[frozenset((c, d))] < pos[key]


def test_create_ex_transport_validation(Q):
    """qva_plan_create_ex rejects a host transport with a missing function before touching a device
    (include/qva.h); a complete one gets as far as the device (no GPU here: a CUDA error)."""
    import ctypes
    d = Q.PlanDesc()
    d.dim, d.n_qubits, d.mixer, d.rank, d.world = 1 << 14, 14, 0, 0, 2
    h = ctypes.c_void_p()
    t = Q.Transport()  # all NULL
    st = Q.lib().qva_plan_create_ex(ctypes.byref(d), ctypes.byref(t), ctypes.byref(h))
    assert st == 1 and not h.value
    assert b"transport" in Q.lib().qva_last_error()


def test_sparse_rows_partition_rule(Q):
    """qva_set_sparse_mixer_rows takes this rank's COMM-psi rows: the host partition rule gives
    contiguous blocks covering [0, dim) with the remainder on the lowest ranks (R16)."""
    for N, world in ((1000, 2), (1000, 4), (1000, 3), (7, 4)):
        parts = [Q.qva_partition(N, world, r) for r in range(world)]
        assert sum(n for n, _ in parts) == N
        assert parts[0][1] == 0
        for (n0, o0), (n1, o1) in zip(parts, parts[1:]):
            assert o1 == o0 + n0 and n0 >= n1
