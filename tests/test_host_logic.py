"""Host-side contract of the drop-in (no GPU needed): the reference's
preconditions raise the reference's exception classes before any compute,
the dtype rule, the filter bank, and that the product has no CPU fallback and
never imports the oracle."""

import ast
import math
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import errors

PKG = Path(wf.__file__).resolve().parent
H, D = wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4


def test_filter_bank_matches_reference_contract():
    """test_wavelet.py:34-59"""
    bank = wf.d4_filters()
    s3, sc = math.sqrt(3.0), 4.0 * math.sqrt(2.0)
    assert np.allclose(bank.analysis_low, [(1 + s3) / sc, (3 + s3) / sc, (3 - s3) / sc,
                                           (1 - s3) / sc], atol=1e-12, rtol=0)
    low, high = bank.analysis_low, bank.analysis_high
    assert bank.synthesis_even.tolist() == [low[2], high[2], low[0], high[0]]
    assert bank.synthesis_odd.tolist() == [low[3], high[3], low[1], high[1]]
    with pytest.raises(ValueError):
        bank.analysis_low[0] = 0.0


def test_transform_preconditions():
    """test_wavelet.py:196-216"""
    with pytest.raises(errors.OddLength):
        wf.dwt1d_forward(np.zeros(5), H)
    with pytest.raises(errors.TooShort):
        wf.dwt1d_forward(np.zeros(0), H)
    with pytest.raises(errors.TooShort):
        wf.dwt1d_forward(np.zeros(2), D)
    with pytest.raises(errors.OddLength):
        wf.dwt1d_inverse(np.zeros(7), D)
    with pytest.raises(errors.OddDimension):
        wf.dwt2d_forward(np.zeros((4, 7)), H)
    with pytest.raises(errors.OddDimension):
        wf.dwt2d_inverse(np.zeros((3, 4)), H)
    with pytest.raises(errors.TooSmall):
        wf.dwt2d_forward(np.zeros((2, 8)), D)
    with pytest.raises(errors.TooSmall):
        wf.dwt2d_forward(np.zeros((0, 0)), H)
    with pytest.raises(ValueError):
        wf.dwt2d_forward(np.zeros(8), H)
    with pytest.raises(ValueError):
        wf.dwt1d_forward(np.zeros((2, 2)), H)


def test_fusion_preconditions():
    """test_fusion.py:161-165, 190-205"""
    with pytest.raises(errors.OddDimension):
        wf.fuse_dwt(np.ones((5, 4)), np.ones((2, 2)), H)
    with pytest.raises(errors.DimensionMismatch):
        wf.fuse_dwt(np.ones((4, 4)), np.ones((3, 2)), H)
    with pytest.raises(ValueError):
        wf.fuse_dwt(np.ones(4), np.ones(2), H)
    with pytest.raises(errors.TooSmall):
        wf.fuse_dwt(np.ones((2, 2)), np.ones((1, 1)), D)
    with pytest.raises(errors.BandCountMismatch):
        wf.fuse(np.ones((4, 4)), [], wf.DwtReplace(H))
    with pytest.raises(errors.DimensionMismatch):
        wf.fuse(np.ones((4, 4)), [np.ones((2, 2)), np.ones((3, 3))], wf.DwtReplace(H))
    with pytest.raises(errors.OddDimension):
        wf.fuse(np.ones((5, 5)), [np.ones((2, 2))], wf.DwtReplace(H))
    with pytest.raises(TypeError):
        wf.fuse(np.ones((4, 4)), [np.ones((2, 2))], object())
    with pytest.raises(ValueError):
        wf.resample_bilinear(np.ones((2, 2)), 0, 4)
    with pytest.raises(ValueError):
        wf.resample_bilinear(np.ones(4), 2, 2)


def test_errors_are_fusion_errors():
    for cls in (errors.OddLength, errors.TooShort, errors.OddDimension, errors.TooSmall,
                errors.DimensionMismatch, errors.BandCountMismatch, errors.NotDivisible,
                errors.ZeroBandMean, errors.TooFewBands):
        assert issubclass(cls, errors.FusionError)


def test_method_names():
    assert wf.method_from_name("hdwt") == wf.DwtReplace(H)
    assert wf.method_from_name("ddwt") == wf.DwtReplace(D)
    with pytest.raises(ValueError):
        wf.method_from_name("nope")


def test_resample_identity_is_a_fresh_copy_on_host():
    """test_fusion.py:23-28 (identity never reaches the device)"""
    p = np.array([[1.0, 2.0], [3.0, 4.0]])
    out = wf.resample_bilinear(p, 2, 2)
    assert np.array_equal(out, p)
    out[0, 0] = 99.0
    assert p[0, 0] == 1.0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        wf.fuse_dwt(np.ones((4, 4), np.float32), np.ones((2, 2), np.float32), H)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        wf.dwt2d_forward(np.ones((4, 4)), H)


def test_product_never_imports_oracle():
    for py in PKG.rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), py
            if isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", py


def test_plan_grid_contract():
    """tiling.py:72-86, 276-285 (test_tiling.py:20-60)"""
    g = wf.plan_grid(64, 32, 4, 2)
    assert (g.pan_tile_w, g.pan_tile_h, g.ms_tile_w, g.ms_tile_h) == (16, 16, 8, 8)
    assert g.tile_count == 8 and g.pan_w == 64 and g.pan_h == 32
    with pytest.raises(errors.NotDivisible):
        wf.plan_grid(30, 30, 4, 4)
    with pytest.raises(errors.OddTile):
        wf.plan_grid(30, 30, 2, 2)
    with pytest.raises(ValueError):
        wf.plan_grid(8, 8, 0, 1)
    assert wf.padded_dims(30, 30, 4, 4) == (32, 32)
    with pytest.raises(errors.DimensionMismatch):
        wf.fuse_tiled(np.ones((8, 8)), [np.ones((4, 4))], wf.DwtReplace(H), g)
    with pytest.raises(ValueError):
        wf.fuse_tiled(np.ones((32, 64)), [np.ones((16, 32))], wf.DwtReplace(H), g, workers=0)


def test_exact_default_switch_logic(monkeypatch):
    """The `exact` keyword defaults to the module switch (WF_EXACT /
    set_exact_default); an explicit True/False always wins."""
    from paper_1803_00737_b200 import fusion

    monkeypatch.setattr(fusion, "_EXACT_DEFAULT", False)
    assert fusion._exact(None) is False and fusion._exact(True) is True
    wf.set_exact_default(True)
    try:
        assert fusion._exact(None) is True and fusion._exact(False) is False
    finally:
        wf.set_exact_default(False)
    assert fusion._exact(None) is False


def test_exact_keyword_validates_before_compute():
    """exact=True keeps the reference's precondition order and exceptions
    (fusion.py:137-147): no GPU is touched before they are raised."""
    with pytest.raises(wf.errors.OddDimension):
        wf.fuse(np.ones((5, 8)), [np.ones((2, 4))], wf.DwtReplace(wf.WaveletKind.HAAR), exact=True)
    with pytest.raises(wf.errors.DimensionMismatch):
        wf.fuse_dwt(np.ones((8, 8)), np.ones((3, 4)), wf.WaveletKind.DAUB4, exact=True)
    with pytest.raises(wf.errors.TooSmall):
        wf.fuse_dwt(np.ones((2, 8)), np.ones((1, 4)), wf.WaveletKind.DAUB4, exact=True)
