"""Host half of the PNM front end (paper_1803_00737_b200/pnm.py): header
parsing and encoding follow imageio.py:22-101 with its exception classes.
The cases restate the reference's own tests (tests/test_imageio.py:13-88 of
the reference package) plus the reference CLI's files in tests/golden/pnm.npz.
No GPU needed: headers never leave the host."""

import numpy as np
import pytest

from paper_1803_00737_b200 import pnm
from paper_1803_00737_b200.errors import FusionError, MalformedHeader, Truncated, UnsupportedFormat
from paper_1803_00737_b200.fusion import DwtReplace
from paper_1803_00737_b200.wavelet import WaveletKind
from oracle import cpu_raster as R


def test_read_pgm_minimal():
    img = pnm.read_pnm(b"P5\n2 2\n255\n" + bytes([0, 64, 128, 255]))
    assert img.dtype == np.uint8 and img.tolist() == [[0, 64], [128, 255]]


def test_read_ppm_minimal():
    img = pnm.read_pnm(b"P6\n2 1\n255\n" + bytes(range(6)))
    assert img.shape == (1, 2, 3)
    assert img[0, 0].tolist() == [0, 1, 2] and img[0, 1].tolist() == [3, 4, 5]


def test_comments_odd_whitespace_and_whitespace_payload():
    img = pnm.read_pnm(b"P5 # a comment\n# another line\n 3\t1 #w h\n255 " + bytes([9, 8, 7]))
    assert img.tolist() == [[9, 8, 7]]
    assert pnm.read_pnm(b"P5\n1 1\n255\n" + bytes([0x20]))[0, 0] == 0x20


@pytest.mark.parametrize("shape", [(13, 17), (5, 9, 3)])
def test_roundtrip(shape):
    img = np.random.default_rng(7).integers(0, 256, size=shape, dtype=np.uint8)
    data = pnm.write_pnm(img)
    assert data == R.encode_pnm(img)
    assert np.array_equal(pnm.read_pnm(data), img)


@pytest.mark.parametrize("data,exc", [
    (b"P4\n2 2\n" + bytes(2), UnsupportedFormat),
    (b"GIF89a", UnsupportedFormat),
    (b"P5\n2 2\n65535\n" + bytes(8), UnsupportedFormat),
    (b"P5\nx 2\n255\n" + bytes(4), MalformedHeader),
    (b"P5\n0 2\n255\n", MalformedHeader),
    (b"P", MalformedHeader),
    (b"P5x2 2\n255\n" + bytes(4), MalformedHeader),
    (b"P5\n2 2 # no newline", MalformedHeader),
    (b"P5\n2 2\n255", MalformedHeader),
    (b"P5\n2 2\n255\n" + bytes(3), Truncated),
])
def test_rejects(data, exc):
    with pytest.raises(exc):
        pnm.read_pnm(data)
    assert issubclass(exc, FusionError)


def test_write_rejects_bad_input():
    with pytest.raises(UnsupportedFormat):
        pnm.write_pnm(np.zeros((2, 2), dtype=np.float32))
    with pytest.raises(UnsupportedFormat):
        pnm.write_pnm(np.zeros((2, 2, 4), dtype=np.uint8))


def test_golden_files_parse(golden_pnm):
    for name in ("rgb", "gray2", "gray1", "rs"):
        data = golden_pnm[f"{name}/pan"].tobytes()
        assert np.array_equal(pnm.read_pnm(data), R.parse_pnm(data))
        for k in golden_pnm.keys():
            if k.startswith(f"{name}/") and "/out" in k:
                out = golden_pnm[k].tobytes()
                r = pnm.PnmRaster.parse(out)
                assert pnm.write_pnm(pnm.read_pnm(out)) == out and r.nbytes == len(out) - r.offset


def test_fuse_pnm_rejects_before_compute(golden_pnm):
    pan = golden_pnm["gray1/pan"].tobytes()
    ppm = golden_pnm["rgb/ms0"].tobytes()
    method = DwtReplace(WaveletKind.HAAR)
    with pytest.raises(ValueError, match="grayscale"):
        pnm.fuse_pnm(ppm, [ppm], method)
    with pytest.raises(ValueError, match="grayscale"):
        pnm.fuse_pnm(pan, [ppm, ppm], method)
    with pytest.raises(Truncated):
        pnm.fuse_pnm(pan, [ppm[:-1]], method)
