"""The C-ABI library: built for sm_100a, loadable, exports every symbol the
public header declares, and rejects bad arguments with the right WF_ERR_*
code before touching the GPU (so these run on a CPU-only host)."""

import ctypes
import subprocess

import pytest

from paper_1803_00737_b200 import _build, _native


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_exports_every_header_symbol(lib):
    names = _native.header_symbols()
    assert len(names) >= 24
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_version_string(lib):
    assert b"sm_100a" in lib.wf_version()


def test_product_library_is_not_the_checked_build(lib):
    """The device-side invariants (WF_CHECKS) are compiled into the separate
    debug library only; the default load is the product build."""
    import os

    if os.environ.get("WF_CHECKED", "") not in ("", "0"):
        pytest.skip("WF_CHECKED set: the checked build is loaded on purpose")
    assert _native.LIB_PATH.name == "libwavefuse_b200.so"
    assert lib.wf_checked_build() == 0


FAKE = 0x1000  # never dereferenced: validation returns first


def _fuse(lib, kind=1, h=8, w=8, nbands=1, ms=True):
    arr = _native.ptr_array([FAKE] * max(nbands, 1))
    return lib.wf_fuse_bands_f32(kind, FAKE, w, arr if ms else None, w // 2, arr, w,
                                 nbands, h, w, None)


def test_validation_codes(lib):
    assert _fuse(lib, kind=3) == 1  # ValueError: unknown kind
    assert _fuse(lib, nbands=0) == 6  # BandCountMismatch
    assert _fuse(lib, h=7) == 2  # OddDimension
    assert _fuse(lib, w=9) == 2
    assert _fuse(lib, kind=2, h=2, w=8) == 3  # TooSmall (D4 min 4)
    assert _fuse(lib, kind=1, h=0, w=0) == 3  # TooSmall (Haar min 2)
    assert _fuse(lib, ms=False) == 1
    assert b"odd" in _native_err(lib, lambda: _fuse(lib, h=7))


def _native_err(lib, call):
    call()
    return lib.wf_last_error()


def test_transform_validation_codes(lib):
    f = lib.wf_dwt2d_forward_f64
    assert f(2, FAKE, 2, FAKE, 2, 2, 8, None) == 3  # TooSmall
    assert f(1, FAKE, 7, FAKE, 7, 4, 7, None) == 2  # OddDimension
    r = lib.wf_dwt_rows_forward_f32
    assert r(1, FAKE, 5, FAKE, 5, 1, 5, None) == 7  # OddLength
    assert r(2, FAKE, 2, FAKE, 2, 1, 2, None) == 8  # TooShort
    assert r(1, FAKE, 0, FAKE, 0, 1, 0, None) == 8
    rs = lib.wf_resample_bilinear_f32
    assert rs(FAKE, 2, 2, 2, FAKE, 0, 4, 0, None) == 1  # ValueError


def test_error_code_mapping():
    from paper_1803_00737_b200 import errors

    with pytest.raises(errors.OddDimension):
        _native.check(2)
    with pytest.raises(errors.TooSmall):
        _native.check(3)
    with pytest.raises(errors.CudaError):
        _native.check(5)
    _native.check(0)


def test_threads_have_private_error_state(lib):
    import threading

    msgs = {}

    def worker(h, key):
        _fuse(lib, h=h)
        msgs[key] = lib.wf_last_error()

    t1 = threading.Thread(target=worker, args=(7, "odd"))
    t2 = threading.Thread(target=worker, args=(9, "odd9"))
    t1.start(), t2.start(), t1.join(), t2.join()
    assert b"x7" in msgs["odd"] and b"x9" in msgs["odd9"]


def test_ctypes_signatures_cover_header(lib):
    for name in _native.header_symbols():
        fn = getattr(lib, name)
        assert fn.restype is not None or name == "wf_ctx_destroy", name
        assert isinstance(fn, ctypes._CFuncPtr)
