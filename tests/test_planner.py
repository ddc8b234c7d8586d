"""Host-side planner / code-generator checks through qc_debug_plan (no GPU)."""
import numpy as np
import pytest

import qcgen
from paper_2303_00123_b200 import qc


def test_debug_symbol_exported():
    for s in qc.DEBUG_EXPORTS:
        assert hasattr(qc.lib(), s)


def test_qft30_plan_shape():
    # 1 KiB rows (rb = 6): 6 free tile bits per pass -> H(0..6), ..., H(21..29)
    st = qc.debug_plan(30, qcgen.qft(30), row_bits=6)
    assert st["gates"] == 480 and st["relabels"] == 15
    assert st["passes"] == 4
    assert st["phase_runs"] > 0
    assert st["blob_bytes"] > 0
    # auto row bits (box transport): narrower rows, 9 free tile bits -> 3 passes
    assert qc.debug_plan(30, qcgen.qft(30))["passes"] == 3


def test_auto_row_bits_follows_the_cost_model():
    """Row bits 0 = auto: the planner tries 3..6 row bits and keeps the plan
    the host cost model prefers -- never more passes than the 1 KiB-row plan,
    and the 137 GB TFXY-33 headline drops from 23 to 17 passes."""
    for n, ops in ((30, qcgen.tfxy(30, 10)), (33, qcgen.tfxy(33, 10)), (33, qcgen.qft(33))):
        auto = qc.debug_plan(n, ops)["passes"]
        wide = qc.debug_plan(n, ops, row_bits=6)["passes"]
        assert auto <= wide
    assert qc.debug_plan(33, qcgen.tfxy(33, 10))["passes"] == 17


def test_tfxy_block_fusion_merges_pair_blocks():
    st = qc.debug_plan(20, qcgen.tfxy(20, 10))
    raw = qc.debug_plan(20, qcgen.tfxy(20, 10), block_fusion=False)
    assert st["gates"] == 1178
    # every pair block (CNOT RX RZ CNOT + adjacent RZ layers) becomes one op
    assert st["blocks"] < raw["blocks"] / 4
    assert st["passes"] <= raw["passes"] + 2


def test_permutation_pairs_cancel_exactly():
    ops = [qcgen.Op("CNOT", (1, 3)), qcgen.Op("CNOT", (1, 3)), qcgen.Op("X", (2,)), qcgen.Op("X", (2,))]
    st = qc.debug_plan(6, ops)
    assert st["blocks"] == 0 and st["passes"] == 0


@pytest.mark.parametrize("n,tile", [(4, 0), (9, 5), (16, 8), (20, 0)])
def test_every_gate_is_planned(n, tile):
    ops = qcgen.random_circuit(n, 150, seed=n)
    st = qc.debug_plan(n, ops, tile_bits=tile, block_fusion=False)
    nonswap = sum(1 for o in ops if o.name != "SWAP")
    assert st["blocks"] == nonswap
    # every non-SWAP gate is encoded exactly once (phase runs absorb several);
    # remap swaps are extra permutation ops
    assert st["fused_ops"] <= nonswap + st["remap_swaps"] and st["fused_ops"] > 0


def test_invalid_ops_rejected():
    with pytest.raises(qc.QCError):
        qc.debug_plan(3, [qcgen.Op("H", (0,))] + [qcgen.Op("CNOT", (1, 2))], tile_bits=2)
    arr = qc.encode_ops([qcgen.Op("CNOT", (1, 2))])
    arr[0]["qubits"][1] = 1
    with pytest.raises(qc.QCError):
        qc.debug_plan(4, arr)


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_jit_codegen_compiles_for_sm100a(prec):
    """Generated specialised kernels compile with NVRTC for sm_100a (all op
    kinds / patterns / predicate sources appear in this mix)."""
    n = 14
    ops = qcgen.random_circuit(n, 120, seed=5) + qcgen.qft(n) + qcgen.tfxy(n, 2)
    st = qc.debug_plan(n, ops, precision=prec, tile_bits=10, compile_jit=True)
    assert st["jit_compiled"] == st["passes"] > 1


@pytest.mark.parametrize("n,prec", [(20, "c128"), (28, "c128"), (33, "c128"), (30, "c64")])
def test_remap_cuts_tfxy_passes(n, prec):
    """Row-bit remap: the nearest-neighbour Trotter circuit needs far fewer
    passes when the row bits may change qubits between passes; the plan ends
    in the layout it started from (restore passes counted in `passes`)."""
    ops = qcgen.tfxy(n, 10)
    rb = 6 if prec == "c128" else 7  # same row geometry for both (auto row bits would differ)
    on = qc.debug_plan(n, ops, precision=prec, row_bits=rb)
    off = qc.debug_plan(n, ops, precision=prec, remap=False, row_bits=rb)
    assert off["remap_swaps"] == 0 and off["restore_passes"] == 0
    assert on["remap_swaps"] > 0
    assert on["passes"] * 2 <= off["passes"], (on, off)
    assert on["restore_passes"] <= 3


def test_remap_off_below_tile():
    # whole state in one tile: no passes to remap between
    st = qc.debug_plan(10, qcgen.tfxy(10, 10))
    assert st["passes"] == 1 and st["remap_swaps"] == 0


def _box_tile_indices(layout, nbits):
    """Tile-local order of the amplitudes the box(es) cover, rebuilt from the
    layout alone: dims ascending, box d covers boxbits[d] bits above
    starts[d]; extra (xmask) bits above dim 4's box, one box per value."""
    starts, boxbits, xmask = layout
    offs = [0]
    for d, w in enumerate(boxbits):
        offs = [o | (i << starts[d]) for i in range(1 << w) for o in offs]
    xs = [0]
    for b in range(32):
        if (xmask >> b) & 1:
            xs = xs + [x | (1 << (starts[4] + b)) for x in xs]
    return sorted(x | o for x in xs for o in offs), len(xs)


@pytest.mark.parametrize("seed", range(12))
def test_box_layout_covers_the_tile_in_local_order(seed):
    """TMA box transport: the decomposition of a random tile bit set T into
    <= 5 tensor-map dims (+ boxes over the bits beyond the 5th run) covers
    exactly the 2^|T| amplitudes of the tile, each once; a tile's local index
    order (ascending physical bits) is the boxes' linear order."""
    rng = np.random.default_rng(seed)
    nbits = int(rng.integers(14, 34))
    for dbl in (True, False):
        for _ in range(20):
            rb = int(rng.integers(1, 7))
            hi = rng.choice(np.arange(rb, nbits), size=12 - rb, replace=False)
            T = (1 << rb) - 1
            for p in hi:
                T |= 1 << int(p)
            lay = qc.debug_box_layout(T, nbits, dbl)
            runs = bin(T & ~(T << 1)).count("1")
            if lay is None:
                assert runs > 5  # only tiles with too many runs fall back
                continue
            starts, boxbits, xmask = lay
            assert len(boxbits) <= 5 and starts[0] == 0 and starts[-1] == nbits
            assert all(w <= (7 if dbl else 8) for w in boxbits[:1]) and all(w <= 8 for w in boxbits)
            idx, nbox = _box_tile_indices(lay, nbits)
            tile = sorted(sum(((x >> j) & 1) << int(p) for j, p in enumerate(b for b in range(nbits) if (T >> b) & 1))
                          for x in range(1 << 12))
            assert idx == tile and nbox <= 16
