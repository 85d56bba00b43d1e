"""Tiled fusion with the reference's per-tile semantics (SURVEY.md 8(f) row
f4) against the reference's own fuse_tiled outputs (tests/golden/tiled.npz,
quantized.npz), plus the reference's tiling tests restated."""

from pathlib import Path

import numpy as np
import pytest

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import errors

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).parent / "golden" / "tiled.npz")
Q8 = np.load(Path(__file__).parent / "golden" / "quantized.npz")
KINDS = {"haar": wf.WaveletKind.HAAR, "daub4": wf.WaveletKind.DAUB4}


@pytest.mark.parametrize("kname", list(KINDS))
def test_fuse_tiled_matches_reference(kname):
    for name in ("g0", "g1", "g2", "g3"):
        pan = G[f"{name}/pan"]
        gw, gh = (int(v) for v in G[f"{name}/grid"])
        nb = sum(1 for k in G.files if k.startswith(f"{name}/ms"))
        ms = [G[f"{name}/ms{b}"] for b in range(nb)]
        grid = wf.plan_grid(pan.shape[1], pan.shape[0], gw, gh)
        got = wf.fuse_tiled(pan, ms, wf.DwtReplace(KINDS[kname]), grid, workers=3)
        for b, o in enumerate(got):
            ref = G[f"{name}/{kname}/out{b}"]
            assert o.dtype == ref.dtype and o.shape == ref.shape
            assert float(np.max(np.abs(o.astype(np.float64) - ref))) <= 1e-3, (name, b)


def test_haar_tiles_equal_untiled_bitwise():
    """test_tiling.py:149-154: Haar never crosses an even tile border."""
    pan = G["g0/pan"]
    ms = [G[f"g0/ms{b}"] for b in range(3)]
    grid = wf.plan_grid(96, 64, 2, 2)
    tiled = wf.fuse_tiled(pan, ms, wf.DwtReplace(KINDS["haar"]), grid)
    whole = wf.fuse(pan, ms, wf.DwtReplace(KINDS["haar"]))
    for a, b in zip(tiled, whole):
        assert np.array_equal(a, b)


def test_d4_differences_confined_to_tile_border_band():
    """test_tiling.py:157-168 / test_acceptance.py:174-212."""
    pan = G["g1/pan"]
    ms = [G[f"g1/ms{b}"] for b in range(2)]
    grid = wf.plan_grid(128, 64, 4, 2)
    tiled = wf.fuse_tiled(pan, ms, wf.DwtReplace(KINDS["daub4"]), grid)
    whole = wf.fuse(pan, ms, wf.DwtReplace(KINDS["daub4"]))
    yy, xx = np.meshgrid(np.arange(64), np.arange(128), indexing="ij")
    dx = np.minimum(xx % 32, 31 - xx % 32)
    dy = np.minimum(yy % 32, 31 - yy % 32)
    dist = np.minimum(dx, dy)
    for a, b in zip(tiled, whole):
        diff = np.abs(a.astype(np.float64) - b)
        assert np.max(diff[dist >= 4]) <= 1e-4
        assert np.max(diff) > 1.0


@pytest.mark.parametrize("kname", list(KINDS))
def test_transfer_8bpp_matches_reference(kname):
    """fuse_tiled(..., transfer_8bpp=True) (tiling.py:238-248) vs the
    reference's own output: byte-exact, Haar and D4."""
    pan = Q8["tiled/pan"]
    ms = [Q8[f"tiled/ms{b}"] for b in range(3)]
    grid = wf.plan_grid(64, 64, 2, 2)
    got = wf.fuse_tiled(pan, ms, wf.DwtReplace(KINDS[kname]), grid, transfer_8bpp=True)
    for b, o in enumerate(got):
        ref = Q8[f"tiled/{kname}/out{b}"]
        assert o.dtype == np.uint8
        assert np.array_equal(o, ref)


def test_8bpp_tiles_aligned_for_the_u8_kernels():
    """64-px tiles take the uint8 window kernels; result equals the float32
    route (the two share the arithmetic)."""
    rng = np.random.default_rng(2)
    pan = rng.integers(0, 256, (128, 256), dtype=np.uint8)
    ms = [rng.integers(0, 256, (64, 128), dtype=np.uint8) for _ in range(2)]
    grid = wf.plan_grid(256, 128, 4, 2)
    for kind in KINDS.values():
        fast = wf.fuse_tiled(pan, ms, wf.DwtReplace(kind), grid, transfer_8bpp=True)
        for r in range(2):
            for c in range(4):
                tile = wf.fuse_quantized(pan[64 * r:64 * r + 64, 64 * c:64 * c + 64],
                                         [m[32 * r:32 * r + 32, 32 * c:32 * c + 32] for m in ms],
                                         wf.DwtReplace(kind))
                for b in range(2):
                    assert np.array_equal(fast[b][64 * r:64 * r + 64, 64 * c:64 * c + 64], tile[b])
