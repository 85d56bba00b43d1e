"""8 bpp path on the GPU: uint8 PAN/MS in, quantised
uint8 out, against the reference's own 8 bpp outputs (tests/golden/
quantized.npz, produced by tiling.fuse_tile_quantized + imageio.quantize).

Tolerance: none -- the bytes equal the reference's. Haar is exact in integer
lanes (all intermediates are multiples of 1/4); D4 (kernel v3) computes in
float32 with a proven error bound and recomputes in float64 every pixel
within 2^-9 of a rounding boundary (tools/u8_error_bound.py). The round-1
kernels (WF_D4_U8=v2 / v1, opt-in) are <= 1 LSB and are checked against
quantize() of the float32 kernel instead."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import _native
from oracle import cpu_dwt as O

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).parent / "golden" / "quantized.npz")
KINDS = {"haar": wf.WaveletKind.HAAR, "daub4": wf.WaveletKind.DAUB4}


def _flips(a, b):
    d = np.abs(a.astype(np.int32) - b.astype(np.int32))
    assert d.max() <= 1
    return int((d > 0).sum())


@pytest.mark.parametrize("kname", list(KINDS))
def test_golden_tiles(kname):
    for k in range(4):
        nb = sum(1 for key in G.files if key.startswith(f"t{k}/ms"))
        pan = G[f"t{k}/pan"]
        ms = [G[f"t{k}/ms{b}"] for b in range(nb)]
        got = wf.fuse_quantized(pan, ms, wf.DwtReplace(KINDS[kname]))
        for b, o in enumerate(got):
            ref = G[f"t{k}/{kname}/out{b}"]
            assert o.dtype == np.uint8 and o.shape == ref.shape
            assert np.array_equal(o, ref), (k, b)
        # the float32 worker computation too (tiling.py:163-172)
        f32 = wf.fuse_tile_quantized(pan, ms, wf.DwtReplace(KINDS[kname]))
        for b, o in enumerate(f32):
            assert o.dtype == np.float32
            _flips(wf.quantize(o), G[f"t{k}/{kname}/out{b}"])


def test_quantize_matches_reference():
    assert np.array_equal(wf.quantize(G["quantize/in"]), G["quantize/out"])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_quantize_dtypes_match_oracle(dtype):
    # half-integers, their float neighbours and out-of-range values: the
    # rounding happens in the plane's own dtype, as numpy does it
    rng = np.random.default_rng(7)
    base = rng.integers(-3, 260, size=(64, 96)).astype(dtype) + dtype(0.5)
    nudge = rng.integers(-1, 2, size=base.shape)
    plane = np.where(nudge < 0, np.nextafter(base, dtype(-np.inf)),
                     np.where(nudge > 0, np.nextafter(base, dtype(np.inf)), base)).astype(dtype)
    got = wf.quantize(plane)
    assert got.dtype == np.uint8
    assert np.array_equal(got, O.quantize(plane))
    t = wf.quantize(torch.from_numpy(plane).cuda())
    assert np.array_equal(t.cpu().numpy(), O.quantize(plane))


@pytest.mark.parametrize("kname", list(KINDS))
def test_tiled_8bpp_pipeline(kname):
    """fuse_tiled(..., transfer_8bpp=True) of the reference (tiling.py:238-248)
    rebuilt from GPU pieces: quantize the inputs, fuse each 2x2 tile with
    fuse_quantized, merge by index."""
    pan = G["tiled/pan"]
    ms = [G[f"tiled/ms{b}"] for b in range(3)]
    pan_u8 = wf.quantize(pan)
    ms_u8 = [wf.quantize(m) for m in ms]
    out = [np.empty((64, 64), np.uint8) for _ in range(3)]
    for r in range(2):
        for c in range(2):
            tile = wf.fuse_quantized(pan_u8[32 * r:32 * r + 32, 32 * c:32 * c + 32],
                                     [m[16 * r:16 * r + 16, 16 * c:16 * c + 16] for m in ms_u8],
                                     wf.DwtReplace(KINDS[kname]))
            for b in range(3):
                out[b][32 * r:32 * r + 32, 32 * c:32 * c + 32] = tile[b]
    for b in range(3):
        assert np.array_equal(out[b], G[f"tiled/{kname}/out{b}"])


def test_u8_haar_saturating_values():
    """The 16-bit-lane Haar kernel at the clamp edges: planes drawn mostly from
    {0, 1, 2, 253, 254, 255} drive every lane to both saturation bounds and
    to the round-down boundaries; bit-exact against the oracle."""
    rng = np.random.default_rng(11)
    H, W, B = 512, 1024, 8
    edge = np.array([0, 1, 2, 3, 252, 253, 254, 255], np.uint8)

    def plane(shape):
        x = rng.integers(0, 256, shape, dtype=np.uint8)
        pick = rng.random(shape) < 0.8
        return np.where(pick, edge[rng.integers(0, edge.size, shape)], x).astype(np.uint8)

    pan = plane((H, W))
    ms = [plane((H // 2, W // 2)) for _ in range(B)]
    got = wf.fuse_quantized(pan, ms, wf.DwtReplace(KINDS["haar"]))
    ref = O.fuse_quantized(pan, ms, "haar")
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


@pytest.mark.parametrize("kname", list(KINDS))
def test_large_u8_scene_vs_oracle(kname):
    """2048 x 4096, 6 bands through the 8 bpp kernels (device tensors and the
    host pipeline's row strips agree bit for bit); against the float64
    oracle (the reference's own sequence on wrapped windows): byte-exact."""
    rng = np.random.default_rng(3)
    H, W, B = 2048, 4096, 6
    pan = rng.integers(0, 256, (H, W), dtype=np.uint8)
    ms = [rng.integers(0, 256, (H // 2, W // 2), dtype=np.uint8) for _ in range(B)]
    kind = KINDS[kname]
    host = wf.fuse_quantized(pan, ms, wf.DwtReplace(kind))
    dev = wf.fuse_quantized(torch.from_numpy(pan).cuda(), [torch.from_numpy(m).cuda() for m in ms],
                            wf.DwtReplace(kind))
    for h_, d_ in zip(host, dev):
        assert np.array_equal(h_, d_.cpu().numpy())
    rows = slice(0, 256)  # oracle on a window (D4 rows wrap: use the windowed oracle)
    if kname == "haar":
        ref = O.fuse_quantized(pan[rows], [m[:128] for m in ms], kname)
        for o, r in zip(host, ref):
            assert np.array_equal(o[rows], r)
    else:
        ref = O.fuse_window(
            lambda r, c: pan[np.ix_(r % H, c % W)].astype(np.float32),
            [lambda r, c, m=m: m[np.ix_(r % (H // 2), c % (W // 2))].astype(np.float32)
             for m in ms], kname, 0, 256, 0, W)
        for o, r in zip(host, ref):
            assert np.array_equal(o[rows], O.quantize(r))


def test_unaligned_widths_fall_back():
    """Widths the 8 bpp kernels do not cover go through the reference-exact
    float64 kernels + quantize: byte-exact too."""
    rng = np.random.default_rng(4)
    pan = rng.integers(0, 256, (20, 36), dtype=np.uint8)
    ms = [rng.integers(0, 256, (10, 18), dtype=np.uint8) for _ in range(2)]
    for kname, kind in KINDS.items():
        got = wf.fuse_quantized(pan, ms, wf.DwtReplace(kind))
        ref = O.fuse_quantized(pan, ms, kname)
        for o, r in zip(got, ref):
            assert np.array_equal(o, r)


@pytest.mark.parametrize("shape,nb", [((8, 1024), 1), ((64, 2080), 3), ((40, 32), 2),
                                      ((130, 4096), 6), ((34, 3104), 8)])
@pytest.mark.parametrize("fix", ["", "all", "ref"])
def test_u8_d4_v3_byte_exact_every_fix_path(shape, nb, fix, monkeypatch):
    """Kernel v3 against the reference's bytes (the oracle's float64 sequence
    + quantize, pinned to reference-generated vectors) on whole planes, with
    its three ways to produce a byte forced in turn: the float32 byte outside
    the flag window (default), every unit recomputed by the float64 fix-up
    (WF_U8_FIX=all: the queued path on short row runs, the queue-overflow
    path on long ones), and every pixel in the reference's own operation
    order (WF_U8_FIX=ref). Partial column bands, 1..8 bands, periodic wrap at
    every edge."""
    if fix:
        monkeypatch.setenv("WF_U8_FIX", fix)
        _native.reload_tuning()
    rng = np.random.default_rng(hash((shape, nb)) % 2**32)
    H, W = shape
    pan = rng.integers(0, 256, (H, W), dtype=np.uint8)
    ms = [rng.integers(0, 256, (H // 2, W // 2), dtype=np.uint8) for _ in range(nb)]
    got = wf.fuse_quantized(torch.from_numpy(pan).cuda(),
                            [torch.from_numpy(x).cuda() for x in ms],
                            wf.DwtReplace(wf.WaveletKind.DAUB4))
    ref = O.fuse_quantized(pan, ms, "daub4")
    for g, r in zip(got, ref):
        assert np.array_equal(g.cpu().numpy(), r)


def test_u8_d4_v3_boundary_heavy_inputs():
    """Inputs that put many fused values on or next to a rounding boundary:
    PAN and MS from a handful of levels (smooth, repetitive scenes) -- many
    more pixels take the fix-up than on random data, and every byte must
    still be the reference's."""
    rng = np.random.default_rng(21)
    H, W, B = 256, 2048, 4
    levels = np.array([0, 64, 127, 128, 200, 255], np.uint8)
    pan = levels[rng.integers(0, levels.size, (H // 8, W // 8))].repeat(8, 0).repeat(8, 1)
    ms = [levels[rng.integers(0, levels.size, (H // 16, W // 16))].repeat(8, 0).repeat(8, 1)
          for _ in range(B)]
    got = wf.fuse_quantized(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
    for g, r in zip(got, O.fuse_quantized(pan, ms, "daub4")):
        assert np.array_equal(g, r)


@pytest.mark.parametrize("shape,nb", [((64, 1024), 1), ((96, 2080), 3), ((130, 16000), 6),
                                      ((34, 3104), 8), ((4, 32), 2)])
@pytest.mark.parametrize("variant", ["v2", "v1"])
def test_u8_d4_equals_quantized_f32_kernel(shape, nb, variant, monkeypatch):
    """The round-1 8 bpp D4 kernels, opt-in (WF_D4_U8=v2: 8 columns per
    thread, row-pair packed; v1: the 4-column kernel) run the f32 kernel's
    expression trees, so their bytes equal quantize() of the f32 kernel's
    output on the same (integer-valued) inputs, bit for bit -- including
    partial column bands (W not a multiple of the CTA's 1024 columns), 1..8
    bands and values far outside [0, 255] before the clamp."""
    monkeypatch.setenv("WF_D4_U8", variant)
    _native.reload_tuning()
    rng = np.random.default_rng(11 + nb)
    H, W = shape
    pan = rng.integers(0, 256, (H, W), dtype=np.uint8)
    ms = [rng.integers(0, 256, (H // 2, W // 2), dtype=np.uint8) for _ in range(nb)]
    m = wf.DwtReplace(wf.WaveletKind.DAUB4)
    got = wf.fuse_quantized(torch.from_numpy(pan).cuda(),
                            [torch.from_numpy(x).cuda() for x in ms], m)
    f32 = wf.fuse(torch.from_numpy(pan.astype(np.float32)).cuda(),
                  [torch.from_numpy(x.astype(np.float32)).cuda() for x in ms], m)
    for g, f in zip(got, f32):
        assert np.array_equal(g.cpu().numpy(), wf.quantize(f.cpu().numpy()))


@pytest.mark.parametrize("kname", list(KINDS))
def test_golden_tiles_exact_mode_bit_exact(kname):
    """exact=True: the 8 bpp path runs the reference's float64 sequence, then
    the quantize -- every golden tile's bytes equal the reference worker's
    (tiling.py:163-172 + imageio.py:115-123), D4 included."""
    for k in range(4):
        nb = sum(1 for key in G.files if key.startswith(f"t{k}/ms"))
        pan = G[f"t{k}/pan"]
        ms = [G[f"t{k}/ms{b}"] for b in range(nb)]
        got = wf.fuse_quantized(pan, ms, wf.DwtReplace(KINDS[kname]), exact=True)
        for b, o in enumerate(got):
            assert np.array_equal(o, G[f"t{k}/{kname}/out{b}"]), (k, b)
        f32 = wf.fuse_tile_quantized(pan, ms, wf.DwtReplace(KINDS[kname]), exact=True)
        for b, o in enumerate(f32):
            assert np.array_equal(wf.quantize(o), G[f"t{k}/{kname}/out{b}"]), (k, b)
