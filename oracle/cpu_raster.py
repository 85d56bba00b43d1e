"""ORACLE — test infrastructure only. Never imported by the product package.

CPU (numpy) restatement of the reference's PNM front end and CLI fuse data
path (paths relative to /root/reference/pkg/src/wavefuse/):
- imageio.py:46-101 PGM/PPM decode/encode, :104-112 to_plane;
- tiling.py:274-310 padded_dims / pad_edge / pad_inputs;
- tiling.py:93-152, 213-273 split -> per-tile fuse -> merge;
- cli.py:113-165 cmd_fuse (load, pad, fuse_tiled, crop, quantize, write).

Pinned against the reference CLI's own output files
(tests/golden/pnm.npz, made by tests/golden/make_golden.py running
`wavefuse fuse`) in tests/test_oracle_pinning.py.
"""

from __future__ import annotations

import numpy as np

from . import cpu_dwt as D


def parse_pnm(data: bytes) -> np.ndarray:
    """imageio.py:46-87 for well-formed input: P5 -> (h, w), P6 -> (h, w, 3).
    Header tokens are separated by whitespace and '#' comment lines; one
    whitespace byte separates maxval from the payload."""
    channels = {b"P5": 1, b"P6": 3}[bytes(data[:2])]
    tokens, pos = [], 2
    while len(tokens) < 3:
        c = data[pos:pos + 1]
        if c.isspace():
            pos += 1
        elif c == b"#":
            pos = data.index(b"\n", pos) + 1
        else:
            end = pos
            while data[end:end + 1].isdigit():
                end += 1
            tokens.append(int(data[pos:end]))
            pos = end
    w, h, maxval = tokens
    assert maxval == 255
    pos += 1
    arr = np.frombuffer(data[pos:pos + w * h * channels], dtype=np.uint8)
    return arr.reshape((h, w) if channels == 1 else (h, w, 3)).copy()


def encode_pnm(r: np.ndarray) -> bytes:
    """imageio.py:90-101"""
    magic = b"P5" if r.ndim == 2 else b"P6"
    return magic + b"\n%d %d\n255\n" % (r.shape[1], r.shape[0]) + r.tobytes()


def to_plane(r: np.ndarray, channel: int = 0) -> np.ndarray:
    """imageio.py:104-112"""
    return (r if r.ndim == 2 else r[:, :, channel]).astype(np.float32)


def padded_dims(w: int, h: int, gw: int, gh: int) -> tuple[int, int]:
    """tiling.py:274-282: round up to multiples of 2 * grid."""
    return -(-w // (2 * gw)) * 2 * gw, -(-h // (2 * gh)) * 2 * gh


def pad_edge(plane: np.ndarray, out_w: int, out_h: int) -> np.ndarray:
    """tiling.py:285-293: replicate the last row and column."""
    h, w = plane.shape
    rows = np.minimum(np.arange(out_h), h - 1)
    cols = np.minimum(np.arange(out_w), w - 1)
    return plane[np.ix_(rows, cols)]


def pad_inputs(pan: np.ndarray, ms, gw: int, gh: int):
    """tiling.py:296-310: bands grow in proportion, rounded up."""
    h, w = pan.shape
    pw, ph = padded_dims(w, h, gw, gh)
    if (pw, ph) == (w, h):
        return pan, list(ms)
    bands = [pad_edge(b, -(-b.shape[1] * pw // w), -(-b.shape[0] * ph // h)) for b in ms]
    return pad_edge(pan, pw, ph), bands


def fuse_tiled(pan: np.ndarray, ms, kind, gw: int, gh: int) -> list[np.ndarray]:
    """tiling.py:213-273 (plain mode): bands to half size globally, then every
    tile fused on its own (per-tile periodic wrap) and merged by index."""
    h, w = pan.shape
    half = [b if b.shape == (h // 2, w // 2) else D.resample_bilinear(b, w // 2, h // 2)
            for b in ms]
    th, tw = h // gh, w // gw
    out = [np.empty_like(pan) for _ in half]
    for r in range(gh):
        for c in range(gw):
            sl = np.s_[r * th:(r + 1) * th, c * tw:(c + 1) * tw]
            msl = np.s_[r * th // 2:(r + 1) * th // 2, c * tw // 2:(c + 1) * tw // 2]
            for k, f in enumerate(D.fuse(pan[sl], [b[msl] for b in half], kind)):
                out[k][sl] = f
    return out


def cli_fuse(pan_pnm: bytes, ms_pnm: list[bytes], kind, gw: int, gh: int) -> list[bytes]:
    """cli.py:147-165 (+ _load_plane/_load_bands/_write_fused, :117-144):
    the bytes of the files `wavefuse fuse` writes."""
    pan = to_plane(parse_pnm(pan_pnm))
    rasters = [parse_pnm(m) for m in ms_pnm]
    if len(rasters) == 1 and rasters[0].ndim == 3:
        bands = [to_plane(rasters[0], c) for c in range(3)]
    else:
        bands = [to_plane(r) for r in rasters]
    h, w = pan.shape
    pan_p, ms_p = pad_inputs(pan, bands, gw, gh)
    fused = fuse_tiled(pan_p, ms_p, kind, gw, gh)
    q = [D.quantize(f[:h, :w]) for f in fused]
    if len(q) == 3:
        return [encode_pnm(np.stack(q, axis=-1))]
    return [encode_pnm(b) for b in q]
