"""Device arithmetic self-tests behind the C ABI.

The kernels divide a 3-vector by one scalar with a shared reciprocal
(tofr_core.h v3_div_shared: the compiler's own FP64 division sequence with the
divisor-only part computed once).  Parity with the reference rests on every
quotient being the correctly rounded a / b, so the self-test compares it bit
for bit with the compiler's division over raw 64-bit patterns (all exponents,
subnormals, inf, NaN) and geometry-range operands."""
from __future__ import annotations

import ctypes as C

import pytest

from paper_2605_11536_b200.api import Renderer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 0x9E3779B9, 12345])
def test_shared_reciprocal_division_bit_exact(seed):
    r = Renderer(0)
    bad = C.c_uint64(123)
    r._check(r._lib.tofr_gpu_selftest_div(r.handle, 1 << 26, seed, C.byref(bad)))
    assert bad.value == 0, f"{bad.value} quotients differ from a / b"
