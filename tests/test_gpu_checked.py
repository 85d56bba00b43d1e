"""The checked build (WF_CHECKS, wf_common.cuh): the same kernels with
device-side invariants of the bulk-copy rings -- each ring slot carries the
index of the load it holds, written by the producer before its copies and
verified by every consumer after its full-barrier wait and again before it
releases the slot, and by the 8 bpp fix-up for the three slots it reads --
plus queue bounds. compute-sanitizer is closed on the GPU pool
(profiles/r02_sanitizer_closed.log); this is the substitute for its
racecheck/synccheck on the mbarrier rings.

* the checked library really checks: its self-test traps (in a subprocess,
  the CUDA context does not survive a trap) and the product library's does not;
* the ring kernels' parity tests pass under it: fused f32/f64/u8 D4 (bulk-copy
  rings, the 8 bpp in-ring fix-up with every fix-up path forced) and the QNR
  scene kernel (tensor-map ring, scoring and fused-pass variants).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1803_00737_b200 import _build

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _checked_lib():
    if not _build.LIB_CHECKED.exists():
        pytest.skip("checked library not built (python -m paper_1803_00737_b200._build --checked)")
    return _build.LIB_CHECKED


def _run(code, checked):
    env = dict(os.environ)
    env["WF_CHECKED"] = "1" if checked else "0"
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=300)


SELFTEST = (
    "import sys; sys.path.insert(0, '.')\n"
    "from paper_1803_00737_b200 import _native\n"
    "lib = _native.load()\n"
    "print('lib', _native.LIB_PATH.name, 'checked', lib.wf_checked_build())\n"
    "print('selftest', lib.wf_check_selftest())\n"
)


def test_checked_selftest_traps():
    _checked_lib()
    r = _run(SELFTEST, checked=True)
    out = r.stdout + r.stderr
    assert "libwavefuse_b200_checked.so checked 1" in out, out
    assert "WF_CHECK failed: x == 1" in out, out
    assert "selftest 0" not in out, out  # the failed invariant surfaced as a CUDA error
    r = _run(SELFTEST, checked=False)
    assert "libwavefuse_b200.so checked 0" in r.stdout and "selftest 0" in r.stdout, r.stdout


def test_ring_kernels_under_checked_build():
    _checked_lib()
    sel = ["tests/test_gpu_quantized.py",
           "tests/test_gpu_parity.py",
           "tests/test_gpu_metrics.py",
           "tests/test_gpu_random_shapes.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider", *sel], cwd=ROOT,
                       env={**os.environ, "WF_CHECKED": "1"}, capture_output=True, text=True,
                       timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "WF_CHECK failed" not in r.stdout + r.stderr, tail
    print(tail.strip().splitlines()[-1])
