"""Bounds-checked device build (failure detection).  The `check`
library variant (`-DTOFR_CHECK=1`, built by `__graft_entry__.build()`) tests
every reservoir-grid item, sparse pool row / chunk plane and shift-queue index
against the range its buffer holds, and traps with the failing site.  Each case
of the sanitizer suite (gated ReSTIR on the wavefront engine, mirror replay,
sparse transient grids with bin reuse and spatial passes, plain deposits,
ellipsoidal sampling, the device BVH build, the reference, the solve -> finish
overlap) runs once under the checked library and once under the product
library in child processes: both must finish, with bit-identical images (the
checks change no arithmetic)."""
from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from tests.test_gpu_sanitizer import _CHILD, CASES

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
CHECK_LIB = ROOT / "paper_2605_11536_b200" / "_native" / "variants" / "libtofr_b200_check.so"


def _run(case: str, extra: dict, lib: Path | None) -> str:
    env = {**os.environ, **extra}
    env.pop("TOFR_B200_LIB", None)
    if lib is not None:
        env["TOFR_B200_LIB"] = str(lib)
    p = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), case], capture_output=True, text=True, env=env,
                       timeout=900)
    log = p.stdout + p.stderr
    assert "TOFR_CHECK failed" not in log, log[-3000:]
    assert p.returncode == 0 and "child ok" in log, log[-3000:]
    return log


_SELFTEST = r"""
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
from paper_2605_11536_b200.api import Renderer
r = Renderer(0)
chk = C.c_int32(-1)
rc = r._lib.tofr_gpu_debug_check_selftest(r.handle, C.byref(chk))
print("selftest rc", rc, "checked", chk.value)
"""


@pytest.mark.parametrize("lib", ["check", "product"])
def test_bounds_check_fires(lib):
    """An out-of-range grid item traps in the checked build and is not
    checked (no memory touched) in the product build."""
    env = {k: v for k, v in os.environ.items() if k != "TOFR_B200_LIB"}
    if lib == "check":
        env["TOFR_B200_LIB"] = str(CHECK_LIB)
    p = subprocess.run([sys.executable, "-c", _SELFTEST, str(ROOT)], capture_output=True, text=True, env=env,
                       timeout=300)
    log = p.stdout + p.stderr
    if lib == "check":
        assert "TOFR_CHECK failed" in log and "i >= s.ilo && i < s.ihi" in log, log[-2000:]
        assert "selftest rc 4" in log, log[-2000:]
    else:
        assert "selftest rc 0 checked 0" in log, log[-2000:]


@pytest.mark.parametrize("name", sorted(CASES))
def test_bounds_checked_build_clean(name):
    if not CHECK_LIB.exists():
        pytest.fail(f"{CHECK_LIB} missing: run __graft_entry__.build()")
    case = name.replace("_overlap", "")
    checked = _run(case, CASES[name], CHECK_LIB)
    plain = _run(case, CASES[name], None)
    h = [re.findall(r"image sha1 (\w+)", x) for x in (checked, plain)]
    assert h[0] == h[1], h
