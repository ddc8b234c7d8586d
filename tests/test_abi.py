"""CPU-side checks of the C-ABI library: it loads and exports every symbol
include/qc.h declares; struct layouts agree with the binding; error paths
work without a GPU.  No compute calls."""
import ctypes
import os
import re

import pytest

import paper_2303_00123_b200 as pkg
from paper_2303_00123_b200 import qc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header="qc.h"):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qc_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for s in ("qc_state_create", "qc_apply_gate", "qc_run_circuit", "qc_state_read"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = pkg.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(qc.EXPORTS) == declared_symbols()
    dbg = declared_symbols("qc_debug.h")
    assert not [x for x in dbg if not hasattr(L, x)]
    assert sorted(qc.DEBUG_EXPORTS) == dbg


def test_version_string():
    assert pkg.version().startswith("qc-b200 1")


def test_gate_struct_layout_matches_header():
    # qc_gate: int32 op, int32 qubits[3], uint32 ctrl_state, uint32 flags,
    # double theta, double m[32]  -> 288 bytes
    assert qc.GATE_DTYPE.itemsize == 288
    assert qc.GATE_DTYPE.fields["theta"][1] == 24
    assert qc.GATE_DTYPE.fields["m"][1] == 32
    # struct sizes / offsets as the C compiler lays out include/qc.h and qc_debug.h
    import subprocess, tempfile
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "qc_debug.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(qc_gate), sizeof(qc_info), offsetof(qc_info, last_flops_per_amp),
         sizeof(qc_plan_stats), offsetof(qc_plan_stats, flops_per_amp), sizeof(qc_mgate),
         offsetof(qc_mgate, ctrl_state), offsetof(qc_mgate, matrix));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        sz = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert sz[0] == qc.GATE_DTYPE.itemsize
    assert sz[1] == ctypes.sizeof(qc.qc_info) and sz[2] == qc.qc_info.last_flops_per_amp.offset
    assert sz[3] == ctypes.sizeof(qc.qc_plan_stats) and sz[4] == qc.qc_plan_stats.flops_per_amp.offset
    assert sz[5] == qc.MGATE_DTYPE.itemsize
    assert sz[6] == qc.MGATE_DTYPE.fields["ctrl_state"][1] and sz[7] == qc.MGATE_DTYPE.fields["matrix"][1]


def test_op_codes_match_header():
    txt = open(os.path.join(ROOT, "include", "qc.h")).read()
    for name, code in qc.OPS.items():
        assert re.search(rf"QC_{name}\s*=\s*{code}\b", txt), name
    assert re.search(rf"QC_MGATE\s*=\s*{qc.QC_MGATE}\b", txt)


def test_encode_generic_gates():
    """MCU records -> QC_MGATE ops indexing a qc_mgate table (matrix pointer
    into a kept-alive complex128 buffer, interleaved re/im, row-major)."""
    import numpy as np
    import qcgen
    rng = np.random.default_rng(0)
    U = qcgen.random_unitary(8, rng)
    ops = [qcgen.Op("H", (0,)), qcgen.Op("MCU", (4, 1, 2, 0, 3), matrix=U, nctrl=2, ctrl_state=2),
           qcgen.Op("MCU", (5,), matrix=np.eye(2), nctrl=0)]
    a = qc.encode_ops(ops)
    assert a[1]["op"] == qc.QC_MGATE and a[1]["qubits"][0] == 0 and a[2]["qubits"][0] == 1
    mt = a.mtab
    assert len(mt) == 2 and mt[0]["n_ctrl"] == 2 and mt[0]["n_targ"] == 3
    assert list(mt[0]["qubits"][:5]) == [4, 1, 2, 0, 3] and mt[0]["ctrl_state"] == 2
    back = np.ctypeslib.as_array(ctypes.cast(int(mt[0]["matrix"]), ctypes.POINTER(ctypes.c_double)),
                                 shape=(128,))
    assert np.array_equal(back[0::2] + 1j * back[1::2], U.reshape(-1))


def test_encode_ops_roundtrip():
    import numpy as np
    import qcgen
    ops = [qcgen.Op("CP", (3, 1), theta=0.25), qcgen.Op("U2", (0, 2), matrix=np.eye(4) * 1j),
           qcgen.Op("CNOT", (1, 2), ctrl_state=0)]
    a = qc.encode_ops(ops)
    assert a[0]["op"] == qc.OPS["CP"] and list(a[0]["qubits"][:2]) == [3, 1]
    assert a[0]["theta"] == 0.25 and a[0]["ctrl_state"] == 1
    assert a[1]["m"][1] == 1.0 and a[1]["m"][0] == 0.0 and a[1]["m"][2 * 5 + 1] == 1.0
    assert a[2]["ctrl_state"] == 0


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU error path")
def test_create_without_gpu_fails_cleanly():
    L = pkg.lib()
    assert L.qc_state_create(10, 1) is None
    assert len(L.qc_last_error()) > 0
    with pytest.raises(qc.QCError):
        pkg.State(5, "c128")


def test_null_state_is_rejected():
    L = pkg.lib()
    assert L.qc_state_sync(None) == qc.QC_ERR_INVALID_ARG
    assert b"NULL" in L.qc_last_error()
    L.qc_state_destroy(None)  # no-op
