"""GPU half of the PNM front end against the
reference: to_plane / pad_edge / pad_inputs against reference-generated
outputs, and fuse_pnm against the files the reference CLI wrote
(`wavefuse fuse`, tests/golden/pnm.npz) -- byte-identical in exact mode."""

import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import pnm, tiling
from paper_1803_00737_b200.errors import ChannelOutOfRange

pytestmark = pytest.mark.gpu

CASES = ("rgb", "gray2", "gray1", "rs")
METHODS = {"hdwt": wf.WaveletKind.HAAR, "ddwt": wf.WaveletKind.DAUB4}


def _inputs(g, name):
    ms = [g[k].tobytes() for k in sorted(k for k in g.keys() if k.startswith(f"{name}/ms"))]
    return g[f"{name}/pan"].tobytes(), ms, tuple(int(v) for v in g[f"{name}/grid"])


def _outputs(g, name, method):
    return [g[k].tobytes() for k in sorted(
        k for k in g.keys() if k.startswith(f"{name}/{method}/out"))]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", list(METHODS))
def test_fuse_pnm_exact_is_byte_identical(golden_pnm, name, method):
    pan, ms, grid = _inputs(golden_pnm, name)
    got = pnm.fuse_pnm(pan, ms, wf.DwtReplace(METHODS[method]), grid, exact=True)
    assert got == _outputs(golden_pnm, name, method)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", list(METHODS))
def test_fuse_pnm_default_byte_identical(golden_pnm, name, method):
    """The default (no `exact` argument) writes the reference CLI's bytes."""
    pan, ms, grid = _inputs(golden_pnm, name)
    got = pnm.fuse_pnm(pan, ms, wf.DwtReplace(METHODS[method]), grid)
    assert got == _outputs(golden_pnm, name, method)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", list(METHODS))
def test_fuse_pnm_fused_kernels(golden_pnm, name, method):
    """exact=False (the fused float32 kernels): same headers and sizes;
    samples within 1 LSB of the reference (a float32 value can round across
    a .5 boundary), and Haar on unresampled 8-bit input is exact (every value
    is a multiple of 1/4)."""
    pan, ms, grid = _inputs(golden_pnm, name)
    got = pnm.fuse_pnm(pan, ms, wf.DwtReplace(METHODS[method]), grid, exact=False)
    want = _outputs(golden_pnm, name, method)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        rg, rw = pnm.PnmRaster.parse(g), pnm.PnmRaster.parse(w)
        assert g[:rg.offset] == w[:rw.offset]
        a = np.frombuffer(g[rg.offset:], np.uint8).astype(int)
        b = np.frombuffer(w[rw.offset:], np.uint8).astype(int)
        assert np.abs(a - b).max() <= 1
        if method == "hdwt" and name != "rs":
            assert np.array_equal(a, b)
        assert np.count_nonzero(a != b) <= max(2, a.size // 1000)


def test_to_plane_gray_color_and_errors():
    gray = np.array([[1, 2], [3, 4]], dtype=np.uint8)
    p = pnm.to_plane(gray)
    assert p.dtype == np.float32 and p.tolist() == [[1.0, 2.0], [3.0, 4.0]]
    color = np.zeros((1, 2, 3), dtype=np.uint8)
    color[0, 0], color[0, 1] = (10, 20, 30), (40, 50, 60)
    assert pnm.to_plane(color, 1).tolist() == [[20.0, 50.0]]
    t = pnm.to_plane(torch.from_numpy(color).cuda(), 2)
    assert t.is_cuda and t.cpu().tolist() == [[30.0, 60.0]]
    for r, c in ((color, 3), (gray, 1), (color, -1)):
        with pytest.raises(ChannelOutOfRange):
            pnm.to_plane(r, c)


def test_read_pnm_device_and_quantize_any_shape(golden_pnm):
    data = golden_pnm["rgb/ms0"].tobytes()
    d = pnm.read_pnm(data, device=True)
    assert d.is_cuda and np.array_equal(d.cpu().numpy(), pnm.read_pnm(data))
    assert pnm.write_pnm(d) == pnm.write_pnm(pnm.read_pnm(data))
    plane = np.array([-3.2, 0.4, 0.5, 127.5, 254.49, 300.0], dtype=np.float32)
    assert pnm.quantize(plane).tolist() == [0, 0, 1, 128, 254, 255]
    img = np.random.default_rng(9).integers(0, 256, size=(16, 16), dtype=np.uint8)
    assert np.array_equal(pnm.quantize(pnm.to_plane(img)), img)


def test_pad_edge_and_pad_inputs_match_reference(golden_pnm):
    for name in ("p0", "p1", "p2"):
        src, want = golden_pnm[f"pad/{name}/in"], golden_pnm[f"pad/{name}/out"]
        got = tiling.pad_edge(src, want.shape[1], want.shape[0])
        assert got.dtype == want.dtype and np.array_equal(got, want)
        t = torch.from_numpy(src).cuda()
        gt = tiling.pad_edge(t, want.shape[1], want.shape[0])
        assert gt.data_ptr() != t.data_ptr() and np.array_equal(gt.cpu().numpy(), want)
    with pytest.raises(ValueError):
        tiling.pad_edge(golden_pnm["pad/p0/in"], 3, 3)
    pan, ms = golden_pnm["padin/pan"], [golden_pnm["padin/ms0"], golden_pnm["padin/ms1"]]
    pp, mp = tiling.pad_inputs(pan, ms, 4, 3)
    assert np.array_equal(pp, golden_pnm["padin/out_pan"])
    assert np.array_equal(mp[0], golden_pnm["padin/out_ms0"])
    assert np.array_equal(mp[1], golden_pnm["padin/out_ms1"])


def test_fuse_tiled_exact_matches_reference_tiles():
    """fuse_tiled(..., exact=True) equals the reference's fuse_tiled bit for
    bit (tests/golden/tiled.npz, recorded with workers=2)."""
    from conftest import Golden
    g = Golden("tiled")
    for name in ("g0", "g1", "g2", "g3"):
        pan = g[f"{name}/pan"]
        ms = [g[k] for k in sorted(k for k in g.keys() if k.startswith(f"{name}/ms"))]
        gw, gh = (int(v) for v in g[f"{name}/grid"])
        grid = wf.plan_grid(pan.shape[1], pan.shape[0], gw, gh)
        for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
            outs = wf.fuse_tiled(pan, ms, wf.DwtReplace(kind), grid, exact=True)
            for b, o in enumerate(outs):
                assert np.array_equal(o, g[f"{name}/{kind.value}/out{b}"])
