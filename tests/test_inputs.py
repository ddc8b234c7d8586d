"""Pins for the seeded input generators (qcgen)."""
import math

import numpy as np

import qcgen


def test_splitmix64_reference_values():
    # First outputs of Vigna's reference splitmix64 seeded with 0.
    out = qcgen.splitmix64(0, np.arange(3, dtype=np.uint64))
    assert [int(x) for x in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                     0x06C45D188009454F]


def test_random_state_recipe():
    n = 10
    s = qcgen.random_state(n)
    assert s.dtype == np.complex128 and s.size == 1 << n
    assert np.all(np.abs(s.real) <= math.sqrt(1.5 / (1 << n)))
    # normalised in expectation: |norm^2 - 1| ~ O(1/sqrt(N))
    assert abs(np.vdot(s, s).real - 1.0) < 0.1
    # chunked generation is identical to whole generation
    part = qcgen.random_state(n, first=100, count=77)
    assert np.array_equal(part, s[100:177])
    c64 = qcgen.random_state(n, precision="c64")
    assert c64.dtype == np.complex64 and np.array_equal(c64, s.astype(np.complex64))


def test_angles_range_and_determinism():
    a = qcgen.angles(1000)
    assert np.all(a >= 0) and np.all(a < 2 * math.pi)
    assert np.array_equal(a, qcgen.angles(1000))
    assert not np.array_equal(a, qcgen.angles(1000, seed=1))


def test_even_parity_state_support():
    n = 6
    s = qcgen.random_state_even_parity(n)
    for i in range(1 << n):
        if bin(i).count("1") & 1:
            assert s[i] == 0
        else:
            assert s[i] != 0
