"""openQASM 2.0 front end (qc_qasm_parse / qc_qasm_emit).

The paper states I/O "through openQASM" (P:6); the grammar, examples and
properties are SPEC S:442-495.  Host-only: these run without a GPU.  The
oracle (test infrastructure) simulates the parsed lists to check that a
round trip keeps the circuit's action.
"""
import math

import numpy as np
import pytest

import oracle
import qcgen
from paper_2303_00123_b200 import qc

HDR = 'OPENQASM 2.0;\ninclude "qelib1.inc";\n'
NAMES = {v: k for k, v in qc.OPS.items()}
SUPPORTED = ("H", "X", "Y", "Z", "P", "RX", "RY", "RZ", "CNOT", "CZ", "CP", "SWAP", "CCX")


def to_ops(arr):
    out = []
    for g in arr:
        name = NAMES[int(g["op"])]
        k = qcgen.ARITY[name]
        th = float(g["theta"]) if name in qcgen.THETA_OPS else None
        out.append(qcgen.Op(name, tuple(int(q) for q in g["qubits"][:k]), theta=th))
    return out


def test_emit_minimal_program():
    assert qc.qasm_emit(1, [qcgen.Op("X", (0,))]) == HDR + "qreg q[1];\nx q[0];\n"


def test_emit_qft2_statements():  # S:462 (build_qft(2), angle -2*pi/4)
    txt = qc.qasm_emit(2, qcgen.qft(2))
    assert txt.splitlines()[3:] == ["h q[0];", "cu1(-1.5707963267948966) q[1],q[0];", "h q[1];",
                                    "swap q[0],q[1];"]


def test_emit_rejects_generic_matrix_and_zero_controls():
    with pytest.raises(qc.QCError):
        qc.qasm_emit(2, [qcgen.Op("U2", (0, 1), matrix=np.eye(4))])
    with pytest.raises(qc.QCError):
        qc.qasm_emit(2, [qcgen.Op("CNOT", (0, 1), ctrl_state=0)])


def test_parse_single_cx():
    n, arr = qc.qasm_parse(HDR + "qreg q[2];\ncx q[0],q[1];\n")
    assert n == 2 and len(arr) == 1
    assert int(arr[0]["op"]) == qc.OPS["CNOT"] and list(arr[0]["qubits"][:2]) == [0, 1]


def test_parse_angle_expression():
    n, arr = qc.qasm_parse(HDR + "qreg q[2];\ncu1(pi/2) q[0],q[1];\n")
    assert int(arr[0]["op"]) == qc.OPS["CP"] and list(arr[0]["qubits"][:2]) == [0, 1]
    assert arr[0]["theta"] == math.pi / 2


def test_parse_expression_grammar_and_aliases():
    txt = HDR + ("qreg r[3]; // comment\r\n"
                 "u1(-(pi - 1)*2/4) r[2]; p(+1.5e-3) r[0]; rz(2*-pi) r[1];\n"
                 "CX r[2],r[0]; cp(.25) r[1],r[2]; ccx r[0],r[1],r[2]; swap r[0],r[2];\n")
    n, arr = qc.qasm_parse(txt)
    ops = to_ops(arr)
    assert n == 3
    assert [o.name for o in ops] == ["P", "P", "RZ", "CNOT", "CP", "CCX", "SWAP"]
    assert ops[0].theta == -(math.pi - 1) * 2 / 4 and ops[1].theta == 1.5e-3 and ops[2].theta == -2 * math.pi
    assert ops[4].theta == 0.25 and ops[5].qubits == (0, 1, 2)


@pytest.mark.parametrize("seed", range(100))
def test_round_trip_random_circuits(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 9))
    ops = qcgen.random_circuit(n, int(rng.integers(1, 100)), seed=seed, kinds=SUPPORTED,
                               random_ctrl_state=False)
    n2, arr = qc.qasm_parse(qc.qasm_emit(n, ops))
    back = to_ops(arr)
    assert n2 == n and len(back) == len(ops)
    for a, b in zip(ops, back):
        assert a.name == b.name and a.qubits == b.qubits
        if a.theta is not None:
            assert b.theta == a.theta  # %.17g is exact for doubles
    if seed < 10:  # the round trip simulates identically (oracle, fp64)
        st = qcgen.random_state(n, seed=seed)
        assert np.abs(oracle.run(n, st, back) - oracle.run(n, st, ops)).max() <= 1e-12


def test_parsed_qft_is_the_fft():
    n = 5
    _, arr = qc.qasm_parse(qc.qasm_emit(n, qcgen.qft(n)))
    st = qcgen.random_state(n, seed=7)
    got = oracle.run(n, st, to_ops(arr))
    assert np.abs(got - np.fft.fft(st, norm="ortho")).max() <= 1e-13


@pytest.mark.parametrize("body,what", [
    ("qreg q[2];\nh q[0]\n", "expected ';'"),
    ("qreg q[2];\nh q[2];\n", "out of range"),
    ("qreg q[2];\nfoo q[0];\n", "unsupported gate"),
    ("qreg q[2];\nh p[0];\n", "unknown register"),
    ("qreg q[2];\nqreg r[2];\n", "second qreg"),
    ("qreg q[2];\ncreg c[2];\n", "unsupported feature"),
    ("qreg q[2];\nmeasure q[0] -> c[0];\n", "unsupported feature"),
    ("qreg q[2];\nbarrier q;\n", "unsupported feature"),
    ("qreg q[2];\nrx(pi/0) q[0];\n", "division by zero"),
    ("qreg q[2];\nrx(theta) q[0];\n", "unknown symbol"),
    ("qreg q[2];\ncx q[1],q[1];\n", "repeated qubit"),
    ("h q[0];\n", "gate before qreg"),
    ("", "no qreg"),
])
def test_parse_rejects_malformed(body, what):
    with pytest.raises(qc.QCError) as e:
        qc.qasm_parse(HDR + body)
    msg = str(e.value)
    assert what in msg
    assert any(c.isdigit() for c in msg.split("qasm", 1)[-1][:6])  # line:col position


def test_parse_rejects_other_versions_and_includes():
    with pytest.raises(qc.QCError):
        qc.qasm_parse('OPENQASM 3.0;\nqreg q[1];\n')
    with pytest.raises(qc.QCError):
        qc.qasm_parse('OPENQASM 2.0;\ninclude "stdgates.inc";\nqreg q[1];\n')
