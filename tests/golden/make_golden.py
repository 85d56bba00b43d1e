"""Generate golden vectors by running the REFERENCE implementation.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference package `wavefuse` (pure Python + numpy, read-only at
/root/reference/pkg/src) and records its outputs on seeded inputs into
tests/golden/*.npz. The reference does not travel to the GPU box, so these
committed fixtures are how the GPU tests (and the oracle pinning tests) see
the reference's exact answers. Re-running this script must reproduce the
files bit for bit (the inputs are seeded).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from wavefuse import fusion, metrics, wavelet  # noqa: E402  (the reference)

OUT = Path(__file__).resolve().parent
HAAR, D4 = wavelet.WaveletKind.HAAR, wavelet.WaveletKind.DAUB4

# (name, h, w, bands, dtype): covers tiny wrap-aliasing shapes (4x4), widths
# with W % 4 == 2, widths spanning several 128-column warp bands with and
# without the vectorised interior, and a float64 case.
FUSION_CASES = [
    ("f4x4", 4, 4, 1, np.float32),
    ("f6x10", 6, 10, 2, np.float32),
    ("f8x12", 8, 12, 1, np.float32),
    ("f16x16", 16, 16, 3, np.float32),
    ("f34x70", 34, 70, 2, np.float32),
    ("f24x392", 24, 392, 3, np.float32),
    ("f40x262", 40, 262, 2, np.float32),
    ("f10x520", 10, 520, 6, np.float32),
    ("d36x264", 36, 264, 2, np.float64),
    ("d10x6", 10, 6, 1, np.float64),
]

TRANSFORM_SHAPES = [(4, 4), (6, 10), (8, 12), (34, 70), (64, 64), (2, 2), (2, 6)]
VECTOR_LENGTHS = [2, 4, 10, 64, 126]
RESAMPLE_CASES = [((3, 5), (7, 11)), ((7, 8), (14, 16)), ((5, 5), (2, 3)), ((4, 4), (4, 8)),
                  ((16, 24), (32, 48))]


def fusion_golden():
    rng = np.random.default_rng(20261018)
    data = {}
    for name, h, w, nb, dt in FUSION_CASES:
        pan = rng.uniform(0.0, 255.0, (h, w)).astype(dt)
        bands = [rng.uniform(0.0, 255.0, (h // 2, w // 2)).astype(dt) for _ in range(nb)]
        data[f"{name}/pan"] = pan
        for b, band in enumerate(bands):
            data[f"{name}/ms{b}"] = band
        for kind in (HAAR, D4):
            if min(h, w) < 4 and kind is D4:
                continue
            outs = fusion.fuse(pan, bands, fusion.DwtReplace(kind))
            for b, o in enumerate(outs):
                data[f"{name}/{kind.value}/out{b}"] = o
    # resampling dispatch: bands not at half size (fusion.py:177-181)
    pan = rng.uniform(0.0, 255.0, (12, 16)).astype(np.float32)
    odd = [rng.uniform(0.0, 255.0, (5, 7)).astype(np.float32) for _ in range(2)]
    data["resamp/pan"] = pan
    for b, band in enumerate(odd):
        data[f"resamp/ms{b}"] = band
    for kind in (HAAR, D4):
        for b, o in enumerate(fusion.fuse(pan, odd, fusion.DwtReplace(kind))):
            data[f"resamp/{kind.value}/out{b}"] = o
    np.savez_compressed(OUT / "fusion.npz", **data)


def transform_golden():
    rng = np.random.default_rng(7)
    data = {}
    for h, w in TRANSFORM_SHAPES:
        for dt in (np.float32, np.float64):
            x = rng.uniform(0.0, 255.0, (h, w)).astype(dt)
            c = rng.uniform(-255.0, 255.0, (h, w)).astype(dt)
            tag = f"{h}x{w}/{np.dtype(dt).name}"
            data[f"{tag}/x"] = x
            data[f"{tag}/c"] = c
            for kind in (HAAR, D4):
                if min(h, w) < wavelet._MIN_LEN[kind]:
                    continue
                data[f"{tag}/{kind.value}/fwd"] = wavelet.dwt2d_forward(x, kind)
                data[f"{tag}/{kind.value}/inv"] = wavelet.dwt2d_inverse(c, kind)
    for n in VECTOR_LENGTHS:
        for dt in (np.float32, np.float64):
            x = rng.uniform(0.0, 255.0, n).astype(dt)
            tag = f"v{n}/{np.dtype(dt).name}"
            data[f"{tag}/x"] = x
            for kind in (HAAR, D4):
                if n < wavelet._MIN_LEN[kind]:
                    continue
                data[f"{tag}/{kind.value}/fwd"] = wavelet.dwt1d_forward(x, kind)
                data[f"{tag}/{kind.value}/inv"] = wavelet.dwt1d_inverse(x, kind)
    for k, ((ih, iw), (oh, ow)) in enumerate(RESAMPLE_CASES):
        for dt in (np.float32, np.float64):
            x = rng.uniform(0.0, 255.0, (ih, iw)).astype(dt)
            tag = f"rs{k}/{np.dtype(dt).name}"
            data[f"{tag}/x"] = x
            data[f"{tag}/out"] = fusion.resample_bilinear(x, ow, oh)
    np.savez_compressed(OUT / "transforms.npz", **data)


def metrics_golden():
    rng = np.random.default_rng(99)
    data = {}
    # q_index on shapes with partial edge blocks and sub-block planes
    for k, (h, w) in enumerate([(33, 70), (40, 40), (16, 16), (64, 96), (31, 65)]):
        a = rng.uniform(0.0, 255.0, (h, w))
        b = a * 0.7 + rng.uniform(0.0, 60.0, (h, w))
        data[f"q{k}/a"] = a
        data[f"q{k}/b"] = b
        data[f"q{k}/q"] = np.float64(metrics.q_index(a, b))
    # degenerate blocks (den == 0): constant and zero-mean blocks
    a = np.full((64, 64), 5.0)
    b = a.copy()
    b[32:, 32:] = 7.0
    b[:32, 32:] = rng.uniform(0, 255, (32, 32))
    data["qdeg/a"], data["qdeg/b"] = a, b
    data["qdeg/q"] = np.float64(metrics.q_index(a, b))
    # full reports on fused scenes
    for k, (size, nb, kind) in enumerate([(64, 3, HAAR), (64, 3, D4), (96, 4, D4), (48, 2, HAAR)]):
        pan = rng.uniform(0.0, 255.0, (size, size)).astype(np.float32)
        ms = [rng.uniform(1.0, 255.0, (size // 2, size // 2)).astype(np.float32)
              for _ in range(nb)]
        fused = fusion.fuse(pan, ms, fusion.DwtReplace(kind))
        rep = metrics.qnr(fused, ms, pan)
        tag = f"rep{k}"
        data[f"{tag}/pan"] = pan
        for b in range(nb):
            data[f"{tag}/ms{b}"] = ms[b]
            data[f"{tag}/fused{b}"] = fused[b]
        data[f"{tag}/ergas"] = np.float64(rep.ergas)
        data[f"{tag}/q_per_band"] = np.array(rep.q_per_band)
        data[f"{tag}/d_lambda"] = np.float64(rep.d_lambda)
        data[f"{tag}/d_s"] = np.float64(rep.d_s)
        data[f"{tag}/qnr"] = np.float64(rep.qnr)
        data[f"{tag}/degrade0"] = metrics.degrade(fused[0], 2)
    np.savez_compressed(OUT / "metrics.npz", **data)


def quantized_golden():
    """8 bpp path: the reference's worker computation on uint8 tiles,
    [quantize(p) for p in fuse_tile_quantized(pan, ms, method)]
    (tiling.py:163-172, 268-269; imageio.py:115-123), plus a whole
    fuse_tiled(..., transfer_8bpp=True) run."""
    from wavefuse import imageio, tiling

    rng = np.random.default_rng(8)
    data = {}
    for k, (h, w, nb) in enumerate([(64, 96, 3), (32, 64, 2), (40, 128, 6), (16, 48, 1)]):
        pan = rng.integers(0, 256, (h, w), dtype=np.uint8)
        ms = [rng.integers(0, 256, (h // 2, w // 2), dtype=np.uint8) for _ in range(nb)]
        data[f"t{k}/pan"] = pan
        for b, m in enumerate(ms):
            data[f"t{k}/ms{b}"] = m
        for kind in (HAAR, D4):
            outs = [imageio.quantize(p)
                    for p in tiling.fuse_tile_quantized(pan, ms, fusion.DwtReplace(kind))]
            for b, o in enumerate(outs):
                data[f"t{k}/{kind.value}/out{b}"] = o
    pan = rng.uniform(0, 255, (64, 64)).astype(np.float32)
    ms = [rng.uniform(0, 255, (32, 32)).astype(np.float32) for _ in range(3)]
    grid = tiling.plan_grid(64, 64, 2, 2)
    data["tiled/pan"] = pan
    for b, m in enumerate(ms):
        data[f"tiled/ms{b}"] = m
    for kind in (HAAR, D4):
        outs = tiling.fuse_tiled(pan, ms, fusion.DwtReplace(kind), grid, transfer_8bpp=True)
        for b, o in enumerate(outs):
            data[f"tiled/{kind.value}/out{b}"] = o
    q = np.array([[-3.0, 0.49, 0.5, 1.5, 2.5], [254.5, 255.2, 300.0, 127.4999, 127.5]],
                 dtype=np.float32)
    data["quantize/in"] = q
    data["quantize/out"] = imageio.quantize(q)
    np.savez_compressed(OUT / "quantized.npz", **data)


def tiled_golden():
    """tiling.fuse_tiled (tiling.py:213-273): per-tile periodic wrap, plain
    (float) mode, including bands that need the global resample first."""
    from wavefuse import tiling

    rng = np.random.default_rng(12)
    data = {}
    cases = [("g0", 64, 96, 3, 2, 2, (32, 48)), ("g1", 64, 128, 2, 4, 2, (32, 64)),
             ("g2", 48, 48, 2, 3, 3, (24, 24)), ("g3", 40, 80, 2, 2, 2, (13, 21))]
    for name, h, w, nb, gw, gh, mshape in cases:
        pan = rng.uniform(0, 255, (h, w)).astype(np.float32)
        ms = [rng.uniform(0, 255, mshape).astype(np.float32) for _ in range(nb)]
        data[f"{name}/pan"] = pan
        data[f"{name}/grid"] = np.array([gw, gh])
        for b, m in enumerate(ms):
            data[f"{name}/ms{b}"] = m
        grid = tiling.plan_grid(w, h, gw, gh)
        for kind in (HAAR, D4):
            outs = tiling.fuse_tiled(pan, ms, fusion.DwtReplace(kind), grid, workers=2)
            for b, o in enumerate(outs):
                data[f"{name}/{kind.value}/out{b}"] = o
    np.savez_compressed(OUT / "tiled.npz", **data)


def _pgm(a: np.ndarray, comment: bytes = b"") -> bytes:
    h, w = a.shape[:2]
    magic = b"P5" if a.ndim == 2 else b"P6"
    return magic + b"\n" + comment + b"%d %d\n255\n" % (w, h) + np.ascontiguousarray(a).tobytes()


def pnm_golden():
    """The reference CLI end to end (cli.main(["fuse", ...]) on temp files):
    PNM inputs -> edge padding -> fuse_tiled -> crop -> quantize -> PNM
    outputs, recorded byte for byte. Also pad_edge / pad_inputs outputs."""
    import tempfile

    from wavefuse import cli, tiling

    rng = np.random.default_rng(5)
    data = {}
    # (name, pan h, pan w, band shapes, one PPM?, grid)
    cases = [("rgb", 50, 70, (25, 35), True, "2x2"),        # padded to 52x72
             ("gray2", 48, 64, (24, 32), False, "1x1"),      # 2 PGM bands -> 2 PGMs
             ("gray1", 40, 66, (20, 33), False, "2x1"),      # 1 band -> 1 PGM
             ("rs", 44, 60, (13, 17), True, "2x2")]          # bands resampled
    with tempfile.TemporaryDirectory() as tmp:
        for name, h, w, bshape, ppm, grid in cases:
            pan = rng.integers(0, 256, (h, w), dtype=np.uint8)
            pan_b = _pgm(pan, b"# pan with a comment\n")
            nb = 3 if ppm else (2 if name == "gray2" else 1)
            bands = [rng.integers(0, 256, bshape, dtype=np.uint8) for _ in range(nb)]
            ms_b = [_pgm(np.stack(bands, axis=-1))] if ppm else [_pgm(b) for b in bands]
            data[f"{name}/pan"] = np.frombuffer(pan_b, np.uint8)
            data[f"{name}/grid"] = np.array([int(v) for v in grid.split("x")])
            for k, m in enumerate(ms_b):
                data[f"{name}/ms{k}"] = np.frombuffer(m, np.uint8)
            (Path(tmp) / "pan.pgm").write_bytes(pan_b)
            ms_paths = []
            for k, m in enumerate(ms_b):
                path = Path(tmp) / f"ms{k}.{'ppm' if ppm else 'pgm'}"
                path.write_bytes(m)
                ms_paths.append(str(path))
            for method in ("hdwt", "ddwt"):
                out = Path(tmp) / f"{name}_{method}.{'ppm' if ppm else 'pgm'}"
                argv = ["fuse", "--pan", str(Path(tmp) / "pan.pgm"), "--method", method,
                        "--grid", grid, "--workers", "2", "--out", str(out)]
                for mp in ms_paths:
                    argv += ["--ms", mp]
                assert cli.main(argv) == 0
                outs = [out] if nb in (1, 3) else [
                    out.with_name(f"{out.stem}_b{k}.pgm") for k in range(nb)]
                for k, o in enumerate(outs):
                    data[f"{name}/{method}/out{k}"] = np.frombuffer(o.read_bytes(), np.uint8)
    for name, (h, w), (ow, oh) in [("p0", (5, 7), (9, 8)), ("p1", (6, 4), (4, 6)),
                                   ("p2", (1, 3), (4, 2))]:
        plane = rng.uniform(0, 255, (h, w)).astype(np.float32)
        data[f"pad/{name}/in"] = plane
        data[f"pad/{name}/out"] = tiling.pad_edge(plane, ow, oh)
    pan = rng.uniform(0, 255, (50, 70)).astype(np.float32)
    ms = [rng.uniform(0, 255, (25, 35)).astype(np.float32), rng.uniform(0, 255, (13, 17))
          .astype(np.float32)]
    pp, mp_ = tiling.pad_inputs(pan, ms, 4, 3)
    data["padin/pan"], data["padin/ms0"], data["padin/ms1"] = pan, ms[0], ms[1]
    data["padin/out_pan"], data["padin/out_ms0"], data["padin/out_ms1"] = pp, mp_[0], mp_[1]
    np.savez_compressed(OUT / "pnm.npz", **data)


if __name__ == "__main__":
    fusion_golden()
    transform_golden()
    metrics_golden()
    quantized_golden()
    tiled_golden()
    pnm_golden()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
