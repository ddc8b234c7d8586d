"""Pins for the CPU oracle against what the paper and the mathematics fix.

Nothing here re-types the oracle's formulas: each test compares the oracle
with an independent construction (numpy.kron / tensor contraction, library
FFT, scipy expm, the paper's printed index tables and closed forms, exact
invariants).  PAPER.md line numbers are cited as P:n.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import qcgen
from qcgen import Op

GOLD = os.path.join(os.path.dirname(__file__), "golden")

# Pauli matrices from the paper's closed forms:
#   X: psi[a]=phi[b], psi[b]=phi[a];  Y: psi[a]=-i phi[b], psi[b]=i phi[a];
#   Z: psi[a]=phi[a], psi[b]=-phi[b].
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PY = np.array([[0, -1j], [1j, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)


def basis(n, k):
    v = np.zeros(1 << n, dtype=complex)
    v[k] = 1.0
    return v


def rstate(n, seed=7):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return v / np.linalg.norm(v)


def apply_by_tensor(n, U, qubits, state):
    """Independent eq:kron application: move the op's qubit axes to the front
    (listed order = most significant), contract with U, move back."""
    k = len(qubits)
    t = state.reshape((2,) * n)           # axis i = qubit i (big-endian, Def. 1)
    t = np.moveaxis(t, list(qubits), list(range(k)))
    sh = t.shape
    t = (U @ t.reshape(1 << k, -1)).reshape(sh)
    t = np.moveaxis(t, list(range(k)), list(qubits))
    return t.reshape(-1)


# ----------------------------------------------------------------- matrices
def test_pauli_matrices_match_paper_closed_forms():
    for name, M in (("X", PX), ("Y", PY), ("Z", PZ)):
        assert np.array_equal(oracle.embed(Op(name, (0,))), M)


@pytest.mark.parametrize("theta", [0.0, 0.3, -1.7, math.pi, 2.9 * math.pi])
def test_rotations_are_exponentials(theta):
    # DESIGN R4: RX = exp(-i t X/2), RY = exp(-i t Y/2), RZ = exp(-i t Z/2).
    for name, S in (("RX", PX), ("RY", PY), ("RZ", PZ)):
        ref = scipy.linalg.expm(-1j * theta / 2 * S)
        assert np.abs(oracle.embed(Op(name, (0,), theta=theta)) - ref).max() < 1e-14
    # P(t) = e^{i t/2} RZ(t) and P(t)|0> = |0>.
    P = oracle.embed(Op("P", (0,), theta=theta))
    RZ = oracle.embed(Op("RZ", (0,), theta=theta))
    assert np.abs(P - np.exp(1j * theta / 2) * RZ).max() < 1e-15
    assert P[0, 0] == 1 and P[1, 0] == 0 and P[0, 1] == 0


def test_hadamard_and_identities():
    H = oracle.embed(Op("H", (0,)))
    assert np.abs(H - (PX + PZ) / math.sqrt(2)).max() < 1e-16
    assert np.abs(H @ PX @ H - PZ).max() < 1e-15
    th = 0.77
    RX = oracle.embed(Op("RX", (0,), theta=th))
    RZ = oracle.embed(Op("RZ", (0,), theta=th))
    assert np.abs(RX - H @ RZ @ H).max() < 1e-15          # RX = H RZ H
    assert np.abs(oracle.embed(Op("RX", (0,), theta=math.pi)) + 1j * PX).max() < 1e-15


def test_swap_matrix_is_paper_matrix():
    # P:921-930 prints the SWAP matrix.
    S = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)
    assert np.array_equal(oracle.embed(Op("SWAP", (0, 1))), S)


@pytest.mark.parametrize("name", list(qcgen.ALL_KINDS))
def test_every_embedded_gate_is_unitary(name):
    rng = np.random.default_rng(3)
    ops = qcgen.random_circuit(3, 1, seed=int(rng.integers(1 << 30)), kinds=[name])
    U = oracle.embed(ops[0])
    assert np.abs(U @ U.conj().T - np.eye(U.shape[0])).max() < 1e-14


# ------------------------------------------------- index tables of the figures
def _tables():
    with open(os.path.join(GOLD, "fig_index_tables.json")) as f:
        return json.load(f)


def test_fig_1q_index_sets():
    """fig:1q: U on qubit q mixes exactly phi[a_j] and phi[b_j]."""
    V = qcgen.random_unitary(2, np.random.default_rng(11))
    for c in _tables()["fig_1q"]["cases"]:
        q = c["q"]
        for a, b in zip(c["a"], c["b"]):
            out = oracle.run(3, basis(3, a), [Op("X", (q,))])
            assert np.array_equal(out, basis(3, b))
            out = oracle.run(3, basis(3, b), [Op("U1", (q,), matrix=V)])
            exp = np.zeros(8, complex)
            exp[a], exp[b] = V[0, 1], V[1, 1]
            assert np.abs(out - exp).max() < 1e-15


def test_fig_ctrl_1q_index_sets():
    """fig:ctrl-1q: only the control-selected half is touched."""
    V = qcgen.random_unitary(2, np.random.default_rng(12))
    for c in _tables()["fig_ctrl_1q"]["cases"]:
        pairs = dict(zip(c["a"], c["b"]))
        touched = set(c["a"]) | set(c["b"])
        for x in range(8):
            out = oracle.run(3, basis(3, x),
                             [Op("CU1", (c["qc"], c["qt"]), matrix=V, ctrl_state=c["ctrl"])])
            if x not in touched:
                assert np.array_equal(out, basis(3, x))
                continue
            a = x if x in pairs else [k for k, v in pairs.items() if v == x][0]
            b = pairs[a]
            col = 0 if x == a else 1
            exp = np.zeros(8, complex)
            exp[a], exp[b] = V[0, col], V[1, col]
            assert np.abs(out - exp).max() < 1e-15
        # CNOT "just swaps half of the elements".
        for a, b in pairs.items():
            out = oracle.run(3, basis(3, a), [Op("CNOT", (c["qc"], c["qt"]), ctrl_state=c["ctrl"])])
            assert np.array_equal(out, basis(3, b))


def test_fig_dctrl_1q_index_sets():
    """fig:dctrl-1q: doubly controlled gate touches only {6,7}."""
    c = _tables()["fig_dctrl_1q"]["cases"][0]
    for x in range(8):
        out = oracle.run(3, basis(3, x), [Op("CCX", tuple(c["qc"]) + (c["qt"],))])
        if x in c["a"]:
            assert np.array_equal(out, basis(3, c["b"][0]))
        elif x in c["b"]:
            assert np.array_equal(out, basis(3, c["a"][0]))
        else:
            assert np.array_equal(out, basis(3, x))


def test_ccx_mixed_ctrl_state_bit_order():
    """Two controls with mixed required states (fig:dctrl-1q, P:948-978,
    generalised per P:942-946: each control is a predicate on its own index
    bit).  qc.h fixes ctrl_state bit t = required state of LISTED control t.
    Brute force on every basis state of n=4, every ordered choice of
    (control0, control1, target): ctrl_state 1 (c0=1, c1=0) and 2 (c0=0, c1=1)
    tell ``<< t`` from ``<< (nc-1-t)``; 0 and 3 are the symmetric cases."""
    n = 4
    for c0 in range(n):
        for c1 in range(n):
            for t in range(n):
                if len({c0, c1, t}) < 3:
                    continue
                for cs in range(4):
                    for x in range(1 << n):
                        bit = lambda q: (x >> (n - 1 - q)) & 1
                        fire = bit(c0) == (cs & 1) and bit(c1) == ((cs >> 1) & 1)
                        y = x ^ (1 << (n - 1 - t)) if fire else x
                        out = oracle.run(n, basis(n, x), [Op("CCX", (c0, c1, t), ctrl_state=cs)])
                        assert np.array_equal(out, basis(n, y)), (c0, c1, t, cs, x)


def test_cnot_listing_order():
    # eq:kron reading: CNOT(c,t) on |c=1,t=0> -> |1,1>.
    for n, c, t in ((2, 0, 1), (2, 1, 0), (4, 3, 1), (5, 0, 4)):
        x = 1 << (n - 1 - c)
        out = oracle.run(n, basis(n, x), [Op("CNOT", (c, t))])
        assert np.array_equal(out, basis(n, x | (1 << (n - 1 - t))))


def test_paper_closed_forms_on_states():
    """X swap, Y, Z and SWAP psi[b]=phi[c] on random states."""
    n = 5
    phi = rstate(n)
    for q in range(n):
        s = 1 << (n - 1 - q)
        a = np.array([i for i in range(1 << n) if not i & s])
        b = a + s
        out = oracle.run(n, phi, [Op("X", (q,))])
        assert np.array_equal(out[a], phi[b]) and np.array_equal(out[b], phi[a])
        out = oracle.run(n, phi, [Op("Y", (q,))])
        assert np.abs(out[a] + 1j * phi[b]).max() < 1e-16
        assert np.abs(out[b] - 1j * phi[a]).max() < 1e-16
        out = oracle.run(n, phi, [Op("Z", (q,))])
        assert np.array_equal(out[a], phi[a]) and np.array_equal(out[b], -phi[b])
    for q0, q1 in ((0, 1), (1, 4), (0, 4), (3, 2)):
        s0, s1 = 1 << (n - 1 - q0), 1 << (n - 1 - q1)
        a = np.array([i for i in range(1 << n) if not (i & s0) and not (i & s1)])
        out = oracle.run(n, phi, [Op("SWAP", (q0, q1))])
        assert np.array_equal(out[a + s0], phi[a + s1])
        assert np.array_equal(out[a + s1], phi[a + s0])
        assert np.array_equal(out[a], phi[a]) and np.array_equal(out[a + s0 + s1], phi[a + s0 + s1])


# ------------------------------------------------------- brute-force Kronecker
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_contiguous_gates_equal_kron(n):
    """eq:kron: psi = (I_l (x) U (x) I_r) phi, explicit Kronecker."""
    rng = np.random.default_rng(100 + n)
    for name in qcgen.ALL_KINDS:
        k = qcgen.ARITY[name]
        if k > n:
            continue
        for q in range(n - k + 1):
            ops = qcgen.random_circuit(k, 1, seed=int(rng.integers(1 << 30)), kinds=[name])
            op = ops[0]
            # listed qubits ascending and contiguous: the plain kron form
            op = Op(op.name, tuple(range(q, q + k)), op.theta, op.matrix, op.ctrl_state)
            U = oracle.embed(op)
            full = np.kron(np.kron(np.eye(1 << q), U), np.eye(1 << (n - q - k)))
            phi = rstate(n, seed=int(rng.integers(1 << 30)))
            out = oracle.run(n, phi, [op])
            assert np.abs(out - full @ phi).max() < 1e-13, (name, q)


@pytest.mark.parametrize("n", [3, 4, 6, 8, 10])
def test_any_qubits_equal_tensor_contraction(n):
    """Non-contiguous / reordered qubits: same operator, axes permuted."""
    rng = np.random.default_rng(200 + n)
    ops = qcgen.random_circuit(n, 60, seed=int(rng.integers(1 << 30)))
    phi = rstate(n, seed=5)
    ref = phi.copy()
    for op in ops:
        ref = apply_by_tensor(n, oracle.embed(op), op.qubits, ref)
    out = oracle.run(n, phi, ops)
    assert np.abs(out - ref).max() < 1e-12


def test_full_matrix_product_small():
    """Dense full_matrix: product of explicit 2^n x 2^n embeddings."""
    n = 4
    ops = qcgen.random_circuit(n, 25, seed=9)
    F = np.eye(1 << n, dtype=complex)
    for op in ops:
        cols = np.stack([apply_by_tensor(n, oracle.embed(op), op.qubits, basis(n, j))
                         for j in range(1 << n)], axis=1)
        F = cols @ F
    phi = rstate(n, 1)
    assert np.abs(oracle.run(n, phi, ops) - F @ phi).max() < 1e-13
    assert np.abs(F @ F.conj().T - np.eye(1 << n)).max() < 1e-13


# ------------------------------------------------------------------ QFT pins
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_qft_paper_sign_is_fft(n):
    """QFT listing (theta=-2pi/2^j) == numpy.fft.fft(norm='ortho')."""
    phi = rstate(n, 30 + n)
    out = oracle.run(n, phi, qcgen.qft(n, sign=-1))
    assert np.abs(out - np.fft.fft(phi, norm="ortho")).max() < 1e-12
    out = oracle.run(n, phi, qcgen.qft(n, sign=+1))
    assert np.abs(out - np.fft.ifft(phi, norm="ortho")).max() < 1e-12


@pytest.mark.parametrize("n", [3, 6, 9])
def test_qft_basis_closed_form(n):
    """North-star closed form: |k> -> sum_j e^{2 pi i j k / 2^n}/sqrt(2^n) |j>."""
    N = 1 << n
    j = np.arange(N)
    for k in (1, 3, N - 1, N // 2 + 1):
        out = oracle.run(n, basis(n, k), qcgen.qft(n, sign=+1))
        ref = np.exp(2j * np.pi * j * k / N) / math.sqrt(N)
        assert np.abs(out - ref).max() < 1e-12
        # the paper's sign gives the conjugate phases (not sign-blind: k != 0)
        out = oracle.run(n, basis(n, k), qcgen.qft(n, sign=-1))
        assert np.abs(out - ref.conj()).max() < 1e-12


@pytest.mark.parametrize("n", [4, 9])
def test_qft_then_inverse_is_identity(n):
    phi = rstate(n, 2)
    c = qcgen.qft(n)
    out = oracle.run(n, phi, c + qcgen.inverse(c))
    assert np.abs(out - phi).max() < 1e-13


def test_qft_gate_counts():
    for n in range(1, 13):
        assert len(qcgen.qft(n)) == n + n * (n - 1) // 2 + n // 2
    c = qcgen.gate_counts(qcgen.qft(30))
    assert c == {"H": 30, "CP": 435, "SWAP": 15}


# ----------------------------------------------------------------- TFXY pins
def test_tfxy_matches_paper_diagram():
    with open(os.path.join(GOLD, "tfxy_n4_s2_wires.json")) as f:
        g = json.load(f)
    ops = qcgen.tfxy(g["n"], g["steps"])
    assert len(ops) == g["total_gates"]
    wires = [[] for _ in range(g["n"])]
    for op in ops:
        if op.name == "CNOT":
            wires[op.qubits[0]].append("C")
            wires[op.qubits[1]].append("T")
        else:
            wires[op.qubits[0]].append(op.name)
    assert wires == g["wires"]


def test_tfxy_counts():
    assert qcgen.gate_counts(qcgen.tfxy(20, 10)) == {"RZ": 608, "RX": 190, "CNOT": 380}
    assert len(qcgen.tfxy(33, 10)) == 1971
    assert qcgen.gate_counts(qcgen.tfxy(33, 10)) == {"RZ": 1011, "RX": 320, "CNOT": 640}
    assert len(qcgen.tfxy(20, 10, variant="block8")) == 1520


@pytest.mark.parametrize("n,steps", [(4, 2), (7, 3), (10, 2)])
def test_tfxy_zero_angles_is_exact_identity(n, steps):
    # rotations become I and CNOT^2 = I; pure moves -> bitwise equal.
    phi = qcgen.random_state(n, seed=4)
    out = oracle.run(n, phi, qcgen.tfxy(n, steps, angle_values=[0.0]))
    assert np.array_equal(out, phi)


@pytest.mark.parametrize("n,steps", [(5, 3), (6, 3), (9, 2)])
def test_tfxy_parity_sector_exact_zeros(n, steps):
    # every pair block preserves Z-parity -> odd-weight amplitudes stay 0.0
    phi = qcgen.random_state_even_parity(n, seed=8)
    out = oracle.run(n, phi, qcgen.tfxy(n, steps))
    w = np.array([bin(i).count("1") & 1 for i in range(1 << n)])
    assert np.all(out[w == 1] == 0.0)
    assert np.abs(np.linalg.norm(out) - np.linalg.norm(phi)) < 1e-13


# ------------------------------------------------------------- invariants
def test_norm_and_inverse_random_circuit():
    n = 8
    phi = rstate(n, 3)
    ops = qcgen.random_circuit(n, 200, seed=21)
    out = oracle.run(n, phi, ops)
    assert abs(np.linalg.norm(out) - 1.0) < 1e-12
    back = oracle.run(n, out, qcgen.inverse(ops))
    assert np.abs(back - phi).max() < 1e-12


def test_thread_count_determinism():
    n = 12
    phi = rstate(n, 4)
    ops = qcgen.random_circuit(n, 50, seed=5)
    a = oracle.run(n, phi, ops, nthreads=1)
    b = oracle.run(n, phi, ops, nthreads=max(2, oracle.max_threads()))
    assert np.array_equal(a, b)


def test_validation_rejects_bad_ops():
    phi = rstate(3)
    with pytest.raises(ValueError):
        oracle.run(3, phi, [Op("H", (3,))])
    with pytest.raises(ValueError):
        oracle.run(3, phi, [Op("CNOT", (1, 1))])
    with pytest.raises(ValueError):
        oracle.run(3, phi, [Op("H", (0,)), Op("P", (0,), theta=float("nan"))])


def test_empty_circuit_and_double_x():
    phi = rstate(4)
    assert np.array_equal(oracle.run(4, phi, []), phi)
    assert np.array_equal(oracle.run(4, phi, [Op("X", (2,)), Op("X", (2,))]), phi)


# ------------------------------------------------- generic gates
def _embedded_mcu(nctrl, k, U, ctrl_state):
    """Independent construction of the generic gate's 2^nq x 2^nq operator over
    its listed qubits (controls first, MSB first): identity except the block
    whose control bits equal ctrl_state, which holds U."""
    nq = nctrl + k
    E = np.eye(1 << nq, dtype=complex)
    cpat = 0
    for t in range(nctrl):  # listed control t = bit nq-1-t of the local index
        cpat |= ((ctrl_state >> t) & 1) << (nq - 1 - t)
    rows = [cpat | r for r in range(1 << k)]
    E[np.ix_(rows, rows)] = U
    return E


@pytest.mark.parametrize("n", [5, 7])
def test_mcu_equals_tensor_contraction(n):
    """Generic gate (every further qubit is one more inserted bit)
    == the embedded operator contracted on the listed axes, any qubit order,
    0..3 controls, 1..4 targets, every ctrl_state pattern drawn at random."""
    rng = np.random.default_rng(100 + n)
    for _ in range(40):
        k = int(rng.integers(1, 5))
        c = int(rng.integers(0, min(3, n - k) + 1))
        qs = tuple(int(q) for q in rng.choice(n, size=k + c, replace=False))
        U = qcgen.random_unitary(1 << k, rng)
        cs = int(rng.integers(1 << c))
        psi = rstate(n, int(rng.integers(1 << 30)))
        out = oracle.run(n, psi, [Op("MCU", qs, matrix=U, nctrl=c, ctrl_state=cs)])
        ref = apply_by_tensor(n, _embedded_mcu(c, k, U, cs), qs, psi)
        assert np.abs(out - ref).max() < 1e-14, (qs, c, cs)


def test_mcu_contiguous_equals_kron():
    """Brute force: listed qubits 0..nq-1 in order -> kron(E, I) (eq:kron)."""
    rng = np.random.default_rng(5)
    n = 6
    for c, k in ((0, 3), (1, 3), (2, 2), (0, 4), (2, 4)):
        U = qcgen.random_unitary(1 << k, rng)
        cs = int(rng.integers(1 << c)) if c else 0
        full = np.kron(_embedded_mcu(c, k, U, cs), np.eye(1 << (n - c - k)))
        psi = rstate(n, 9 + c + k)
        out = oracle.run(n, psi, [Op("MCU", tuple(range(c + k)), matrix=U, nctrl=c, ctrl_state=cs)])
        assert np.abs(out - full @ psi).max() < 1e-14


def test_fig_dctrl_1q_generic_u():
    """fig:dctrl-1q with a generic U: only phi[6], phi[7] change,
    by exactly U (the doubly controlled gate "touches a quarter")."""
    c = _tables()["fig_dctrl_1q"]["cases"][0]
    V = qcgen.random_unitary(2, np.random.default_rng(21))
    a, b = c["a"][0], c["b"][0]
    for x in range(8):
        out = oracle.run(3, basis(3, x), [Op("MCU", tuple(c["qc"]) + (c["qt"],), matrix=V, nctrl=2)])
        if x == a or x == b:
            col = 0 if x == a else 1
            exp = np.zeros(8, complex)
            exp[a], exp[b] = V[0, col], V[1, col]
            assert np.abs(out - exp).max() < 1e-15
        else:
            assert np.array_equal(out, basis(3, x))


def test_mcu_special_cases_and_inverse():
    """MCU reduces to the named gates (U1, CU1 with either control state, CCX
    with X, U2) and MCU followed by its adjoint is the identity (unitarity)."""
    rng = np.random.default_rng(8)
    n = 5
    psi = rstate(n, 3)
    V = qcgen.random_unitary(2, rng)
    W = qcgen.random_unitary(4, rng)
    pairs = [
        (Op("U1", (2,), matrix=V), Op("MCU", (2,), matrix=V, nctrl=0)),
        (Op("CU1", (4, 1), matrix=V, ctrl_state=0), Op("MCU", (4, 1), matrix=V, nctrl=1, ctrl_state=0)),
        (Op("CU1", (0, 3), matrix=V), Op("MCU", (0, 3), matrix=V, nctrl=1)),
        (Op("U2", (3, 1), matrix=W), Op("MCU", (3, 1), matrix=W, nctrl=0)),
    ] + [(Op("CCX", (1, 4, 2), ctrl_state=cs), Op("MCU", (1, 4, 2), matrix=PX, nctrl=2, ctrl_state=cs))
         for cs in range(4)]
    for named, gen in pairs:
        assert np.array_equal(oracle.run(n, psi, [named]), oracle.run(n, psi, [gen]))
    ops = qcgen.random_mcu_circuit(n, 30, seed=4, p_mcu=1.0)
    back = oracle.run(n, oracle.run(n, psi, ops), qcgen.inverse(ops))
    assert np.abs(back - psi).max() < 1e-13


def test_mcu_validation():
    psi = rstate(4, 1)
    with pytest.raises(ValueError):
        Op("MCU", (0, 1), matrix=np.eye(2), nctrl=0)      # 1 target needs 2x2? -> 2 targets need 4x4
    with pytest.raises(ValueError):
        Op("MCU", (0, 1, 2, 3, 4), matrix=np.eye(32), nctrl=0)  # > 4 targets
    bad = Op("MCU", (0, 1), matrix=np.eye(2), nctrl=1)
    bad.qubits = (0, 0)
    with pytest.raises(ValueError):
        oracle.run(4, psi, [bad])
