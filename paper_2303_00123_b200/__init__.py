"""B200-native state-vector gate engine (hot path of qclab++, arXiv 2303.00123).

The product is the C-ABI library ``libqc.so`` (include/qc.h), built from
``csrc/`` for sm_100a.  :mod:`.qc` is the thin ctypes binding.  There is no
CPU fallback: without the built library every call raises.
"""
from .qc import State, QCError, encode_ops, lib, version, EXPORTS  # noqa: F401

__all__ = ["State", "QCError", "encode_ops", "lib", "version", "EXPORTS"]
