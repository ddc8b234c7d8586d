"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: no gate matrices, no index
masks, no state update.  It only produces
  * initial states (counter-based splitmix64),
  * angles (splitmix64, U[0, 2*pi)),
  * gate lists (the paper's benchmark circuits and random test circuits) as
    plain records ``Op(name, qubits, theta, matrix, ctrl_state)``.

Both sides consume these records and build their own gate matrices:
``oracle/`` in plain C, the product library in its own host C++.

Citations (PAPER.md line numbers, "P:n"):
  * QFT builder  -- Fig. ``fig:MatlabvCpp`` listing, P:353-376 (theta at P:366).
  * TFXY builder -- Fig. ``fig:bm-circ`` (b); reading in DESIGN.md R8.
  * Qubit numbering follows Definition 1: qubit 0 is the MSB.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "GOLDEN", "splitmix64", "u_pm1", "random_state", "random_state_even_parity",
    "angles", "Op", "ARITY", "NCTRL", "qft", "tfxy", "inverse", "random_circuit",
    "random_unitary", "gate_counts", "STATE_SEED", "ANGLE_SEED", "random_mcu_circuit",
    "MCU_MAX_QUBITS", "MCU_MAX_TARGETS",
]

STATE_SEED = 12345
ANGLE_SEED = 67890

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, ctr) -> np.ndarray:
    """Counter-based splitmix64: output #ctr of the stream started at ``seed``.

    x = seed + (ctr+1)*GOLDEN (mod 2^64), then the standard splitmix64 finaliser.
    For seed=0, ctr=0 this is the first output of Vigna's reference splitmix64
    (0xE220A8397B1DCDAF); tests/test_inputs.py pins that.
    """
    c = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def u_pm1(x: np.ndarray) -> np.ndarray:
    """Map 64 random bits to a double in [-1, 1): (x>>11)*2^-52 - 1 (exact)."""
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def _state_scale(n: int) -> float:
    # E[re^2 + im^2] = 2/3 for u ~ U[-1,1), so sqrt(1.5 / 2^n) normalises in
    # expectation; 1.5/2^n is exact and sqrt is correctly rounded, so the scale
    # is bit-identical wherever it is computed (host here, device in K9).
    return math.sqrt(1.5 / float(1 << n))


def random_state(n: int, seed: int = STATE_SEED, precision: str = "c128",
                 first: int = 0, count: Optional[int] = None) -> np.ndarray:
    """Random state amplitudes [first, first+count) of the n-qubit recipe.

    re_i = u(sm(seed, 2i)) * scale, im_i = u(sm(seed, 2i+1)) * scale.
    c64: the double value rounded to float32 (the oracle then starts from the
    exact up-cast).  The state is normalised in expectation, not exactly;
    every parity check is linear in the state, and norm tests compare
    before/after.
    """
    N = 1 << n
    if count is None:
        count = N - first
    i = np.arange(first, first + count, dtype=np.uint64)
    s = _state_scale(n)
    re = u_pm1(splitmix64(seed, np.uint64(2) * i)) * s
    im = u_pm1(splitmix64(seed, np.uint64(2) * i + np.uint64(1))) * s
    out = re + 1j * im
    if precision == "c64":
        return out.astype(np.complex64)
    if precision != "c128":
        raise ValueError(precision)
    return out


def random_state_even_parity(n: int, seed: int = STATE_SEED) -> np.ndarray:
    """Random state supported only on even-Hamming-weight indices (TFXY pin)."""
    st = random_state(n, seed)
    idx = np.arange(1 << n, dtype=np.uint64)
    par = np.zeros(1 << n, dtype=np.uint64)
    for b in range(n):
        par ^= (idx >> np.uint64(b)) & np.uint64(1)
    st[par == 1] = 0
    return st


def angles(count: int, seed: int = ANGLE_SEED) -> np.ndarray:
    """count angles ~ U[0, 2*pi) from splitmix64 (slot order)."""
    x = splitmix64(seed, np.arange(count, dtype=np.uint64))
    u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return u * (2.0 * math.pi)


# ---------------------------------------------------------------- gate records
ARITY = {"H": 1, "X": 1, "Y": 1, "Z": 1, "P": 1, "RX": 1, "RY": 1, "RZ": 1,
         "CNOT": 2, "CZ": 2, "CP": 2, "SWAP": 2, "U1": 1, "CU1": 2, "U2": 2,
         "CCX": 3}
NCTRL = {"CNOT": 1, "CZ": 1, "CP": 1, "CU1": 1, "CCX": 2}
THETA_OPS = {"P", "RX", "RY", "RZ", "CP"}
MATRIX_DIM = {"U1": 2, "CU1": 2, "U2": 4}


# "MCU": the generic gate of SURVEY 8(f) rows 1-2 -- ``nctrl``
# controls listed first, then k = len(qubits) - nctrl targets carrying a dense
# 2^k x 2^k ``matrix`` (big-endian over the listed targets, eq:kron).
MCU_MAX_QUBITS = 16
MCU_MAX_TARGETS = 4


@dataclass
class Op:
    """One gate application.  ``qubits`` lists controls first."""
    name: str
    qubits: Tuple[int, ...]
    theta: Optional[float] = None
    matrix: Optional[np.ndarray] = None
    ctrl_state: Optional[int] = None  # bit t = required state of control t
    nctrl: Optional[int] = None       # MCU only: number of leading control qubits

    def __post_init__(self):
        self.qubits = tuple(int(q) for q in self.qubits)
        if self.name == "MCU":
            nq = len(self.qubits)
            if self.nctrl is None or not (0 <= self.nctrl < nq <= MCU_MAX_QUBITS):
                raise ValueError("MCU needs 0 <= nctrl < len(qubits) <= 16")
            k = nq - self.nctrl
            if k > MCU_MAX_TARGETS:
                raise ValueError("MCU takes at most 4 target qubits")
            m = np.asarray(self.matrix, dtype=np.complex128)
            if m.shape != (1 << k, 1 << k):
                raise ValueError(f"MCU with {k} targets needs a {1 << k}x{1 << k} matrix")
            self.matrix = m
            if self.ctrl_state is None:
                self.ctrl_state = (1 << self.nctrl) - 1
            return
        if self.name not in ARITY:
            raise ValueError(f"unknown op {self.name}")
        if len(self.qubits) != ARITY[self.name]:
            raise ValueError(f"{self.name} takes {ARITY[self.name]} qubits")
        if self.ctrl_state is None:
            self.ctrl_state = (1 << NCTRL.get(self.name, 0)) - 1
        if self.name in THETA_OPS and self.theta is None:
            raise ValueError(f"{self.name} needs theta")
        if self.name in MATRIX_DIM:
            d = MATRIX_DIM[self.name]
            m = np.asarray(self.matrix, dtype=np.complex128)
            if m.shape != (d, d):
                raise ValueError(f"{self.name} needs a {d}x{d} matrix")
            self.matrix = m


def qft(n: int, sign: int = -1) -> List[Op]:
    """QFT exactly as the listing P:353-376 builds it (theta = sign*2*pi/2^j).

    sign=-1 is the paper's listing and equals numpy.fft.fft(norm=
    "ortho"); sign=+1 is the north star's closed form (= ifft).  DESIGN R5.
    """
    if n < 1:
        raise ValueError("n >= 1")
    ops: List[Op] = []
    for i in range(n):
        ops.append(Op("H", (i,)))
        for j in range(2, n - i + 1):
            ctrl = j + i - 1
            th = sign * 2.0 * math.pi / float(1 << j)
            ops.append(Op("CP", (ctrl, i), theta=th))
    for i in range(n // 2):
        ops.append(Op("SWAP", (i, n - i - 1)))
    return ops


def _tfxy_halfsteps(n: int, steps: int):
    even = [(q, q + 1) for q in range(0, n - 1, 2)]
    odd = [(q, q + 1) for q in range(1, n - 1, 2)]
    hs = []
    for _ in range(steps):
        hs.append(even)
        if odd:
            hs.append(odd)
    return hs


def tfxy(n: int, steps: int, seed: int = ANGLE_SEED, variant: str = "literal",
         angle_values: Optional[Sequence[float]] = None) -> List[Op]:
    """1D nearest-neighbour TFXY Trotter circuit, Fig. fig:bm-circ(b) P:89-99.

    variant="literal" (DESIGN R8, default): half-steps alternate even pairs
    (0,1),(2,3),... and odd pairs (1,2),(3,4),...; each pair (q,q+1) gets
    CNOT(q->q+1), RX(q), RZ(q+1), CNOT(q->q+1); RZ layers sit before the first
    half-step (its qubits), between half-steps (union of both), after the
    last (its qubits).  42 gates at n=4, steps=2, matching the diagram.
    variant="block8": SPEC's unmerged 8-gate block per pair.
    One angle per RZ/RX slot, in emission order.
    """
    if n < 2 or steps < 1:
        raise ValueError("n >= 2, steps >= 1")
    slots: List[Tuple[str, Tuple[int, ...]]] = []
    hs = _tfxy_halfsteps(n, steps)
    if variant == "literal":
        def qubits_of(h):
            return sorted({q for p in h for q in p})
        for k, h in enumerate(hs):
            if k == 0:
                layer = qubits_of(h)
            else:
                layer = sorted(set(qubits_of(hs[k - 1])) | set(qubits_of(h)))
            slots += [("RZ", (q,)) for q in layer]
            for (a, b) in h:
                slots += [("CNOT", (a, b)), ("RX", (a,)), ("RZ", (b,)), ("CNOT", (a, b))]
        slots += [("RZ", (q,)) for q in qubits_of(hs[-1])]
    elif variant == "block8":
        for h in hs:
            for (a, b) in h:
                slots += [("RZ", (a,)), ("RZ", (b,)), ("CNOT", (a, b)), ("RX", (a,)),
                          ("RZ", (b,)), ("CNOT", (a, b)), ("RZ", (a,)), ("RZ", (b,))]
    else:
        raise ValueError(variant)
    n_ang = sum(1 for s in slots if s[0] != "CNOT")
    th = np.asarray(angles(n_ang, seed) if angle_values is None else angle_values,
                    dtype=np.float64)
    if th.size == 1 and n_ang > 1:
        th = np.full(n_ang, float(th.reshape(-1)[0]))
    ops: List[Op] = []
    k = 0
    for name, qs in slots:
        if name == "CNOT":
            ops.append(Op("CNOT", qs))
        else:
            ops.append(Op(name, qs, theta=float(th[k])))
            k += 1
    return ops


def inverse(ops: Sequence[Op]) -> List[Op]:
    """Reversed list, each gate replaced by its adjoint (verification aid)."""
    out = []
    for op in reversed(ops):
        if op.name in THETA_OPS:
            out.append(Op(op.name, op.qubits, theta=-op.theta, ctrl_state=op.ctrl_state))
        elif op.name in MATRIX_DIM or op.name == "MCU":
            out.append(Op(op.name, op.qubits, matrix=op.matrix.conj().T.copy(),
                          ctrl_state=op.ctrl_state, nctrl=op.nctrl))
        else:  # H X Y Z CNOT CZ SWAP CCX are self-inverse
            out.append(Op(op.name, op.qubits, ctrl_state=op.ctrl_state))
    return out


def random_unitary(d: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-ish random d x d unitary (QR of a complex Gaussian, phase-fixed)."""
    z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


ALL_KINDS = ("H", "X", "Y", "Z", "P", "RX", "RY", "RZ", "CNOT", "CZ", "CP",
             "SWAP", "U1", "CU1", "U2", "CCX")


def random_circuit(n: int, n_gates: int, seed: int = 1,
                   kinds: Sequence[str] = ALL_KINDS,
                   random_ctrl_state: bool = True) -> List[Op]:
    """Random gate list over ``kinds`` with random (distinct, any-order) qubits."""
    rng = np.random.default_rng(seed)
    kinds = [k for k in kinds if ARITY[k] <= n]
    ops = []
    for _ in range(n_gates):
        name = kinds[rng.integers(len(kinds))]
        qs = tuple(int(q) for q in rng.choice(n, size=ARITY[name], replace=False))
        nc = NCTRL.get(name, 0)
        cs = int(rng.integers(1 << nc)) if (random_ctrl_state and nc) else None
        th = float(rng.uniform(-2 * math.pi, 2 * math.pi)) if name in THETA_OPS else None
        m = random_unitary(MATRIX_DIM[name], rng) if name in MATRIX_DIM else None
        ops.append(Op(name, qs, theta=th, matrix=m, ctrl_state=cs))
    return ops


def random_mcu_circuit(n: int, n_gates: int, seed: int = 1, max_ctrl: int = 4, max_targ: int = 4,
                       mix: Sequence[str] = ALL_KINDS, p_mcu: float = 0.5,
                       perm_frac: float = 0.0) -> List[Op]:
    """Random circuit mixing generic MCU gates (random control count
    0..max_ctrl, target count 1..max_targ, random ctrl_state, Haar-ish matrix;
    with probability perm_frac a random permutation matrix -- a pure move)
    with the named kinds of ``mix``."""
    rng = np.random.default_rng(seed)
    named = random_circuit(n, n_gates, seed=seed + 7919, kinds=mix)
    ops = []
    for i in range(n_gates):
        if rng.random() >= p_mcu:
            ops.append(named[i])
            continue
        k = int(rng.integers(1, min(max_targ, n) + 1))
        c = int(rng.integers(0, min(max_ctrl, n - k) + 1))
        qs = tuple(int(q) for q in rng.choice(n, size=k + c, replace=False))
        if rng.random() < perm_frac:
            m = np.eye(1 << k, dtype=np.complex128)[rng.permutation(1 << k)]
        else:
            m = random_unitary(1 << k, rng)
        ops.append(Op("MCU", qs, matrix=m, nctrl=c, ctrl_state=int(rng.integers(1 << c))))
    return ops


def gate_counts(ops: Sequence[Op]) -> dict:
    c: dict = {}
    for o in ops:
        c[o.name] = c.get(o.name, 0) + 1
    return c
