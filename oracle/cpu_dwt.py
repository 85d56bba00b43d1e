"""ORACLE — test infrastructure only. Never imported by the product package.

CPU (numpy, float64) restatement of the reference's DWT pan-sharpening path,
used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg as the checker. Each function cites the reference code it
restates (paths relative to /root/reference/pkg/src/wavefuse/).

Pinning: tests/test_oracle_pinning.py checks every function here against
golden vectors produced by the reference itself (tests/golden/make_golden.py
imports /root/reference/pkg/src/wavefuse and records its outputs) and against
the reference's own known-answer tests.

The restatement is deliberately written differently from the reference
(explicit periodic index vectors + fancy indexing instead of roll/concatenate)
but performs the same IEEE float64 operations in the same order, so the
outputs are bit-identical to the reference (checked by the pinning tests).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HAAR = "haar"
DAUB4 = "daub4"
_MIN = {HAAR: 2, DAUB4: 4}  # wavelet.py:66
_GAIN = {HAAR: 1.0, DAUB4: 2.0}  # fusion.py:125


def kind_name(kind) -> str:
    """Accept 'haar'/'daub4', the WaveletKind enum of either package, or the
    wire codes 1/2."""
    if isinstance(kind, str):
        return kind
    if isinstance(kind, int):
        return {1: HAAR, 2: DAUB4}[kind]
    return kind.value


def taps():
    """wavelet.py:48-63: h (analysis low), g = QMF mirror, synthesis quads."""
    r3 = math.sqrt(3.0)
    den = 4.0 * math.sqrt(2.0)
    h = [(1.0 + r3) / den, (3.0 + r3) / den, (3.0 - r3) / den, (1.0 - r3) / den]
    g = [h[3], -h[2], h[1], -h[0]]
    even = [h[2], g[2], h[0], g[0]]
    odd = [h[3], g[3], h[1], g[1]]
    return h, g, even, odd


def out_dtype(arr):
    """wavelet.py:69-70 / fusion.py:46-47"""
    return np.float32 if np.asarray(arr).dtype == np.float32 else np.float64


def _quad(f, a, b, c, d):
    # ((f0*a + f1*b) + f2*c) + f3*d, one rounding per op (wavelet.py:85-86)
    return f[0] * a + f[1] * b + f[2] * c + f[3] * d


def analysis_last(x: np.ndarray, kind: str) -> np.ndarray:
    """_forward_last (wavelet.py:73-87) on a float64 array: approximations
    then details along the last axis, periodic wrap."""
    n = x.shape[-1]
    half = n // 2
    ev = np.arange(half) * 2
    e, o = x[..., ev], x[..., ev + 1]
    out = np.empty_like(x)
    if kind == HAAR:
        out[..., :half] = (e + o) * 0.5
        out[..., half:] = (e - o) * 0.5
        return out
    h, g, _, _ = taps()
    nxt = (ev + 2) % n
    e1, o1 = x[..., nxt], x[..., nxt + 1]
    out[..., :half] = _quad(h, e, o, e1, o1)
    out[..., half:] = _quad(g, e, o, e1, o1)
    return out


def synthesis_last(c: np.ndarray, kind: str) -> np.ndarray:
    """_inverse_last (wavelet.py:90-109): rebuild even/odd samples from the
    current (approx, detail) pair and its periodic predecessor."""
    n = c.shape[-1]
    half = n // 2
    a, d = c[..., :half], c[..., half:]
    out = np.empty_like(c)
    if kind == HAAR:
        out[..., 0::2] = a + d
        out[..., 1::2] = a - d
        return out
    _, _, se, so = taps()
    prev = (np.arange(half) - 1) % half
    ap, dp = a[..., prev], d[..., prev]
    out[..., 0::2] = _quad(se, ap, dp, a, d)
    out[..., 1::2] = _quad(so, ap, dp, a, d)
    return out


def dwt1d_forward(x, kind) -> np.ndarray:
    """wavelet.py:131-139"""
    arr = np.asarray(x)
    k = kind_name(kind)
    return analysis_last(arr.astype(np.float64), k).astype(out_dtype(arr))


def dwt1d_inverse(c, kind) -> np.ndarray:
    """wavelet.py:142-146"""
    arr = np.asarray(c)
    k = kind_name(kind)
    return synthesis_last(arr.astype(np.float64), k).astype(out_dtype(arr))


def dwt2d_forward(plane, kind) -> np.ndarray:
    """wavelet.py:149-155: rows, then columns (via the transpose)."""
    arr = np.asarray(plane)
    k = kind_name(kind)
    rows = analysis_last(arr.astype(np.float64), k)
    both = analysis_last(np.ascontiguousarray(rows.T), k).T
    return np.ascontiguousarray(both).astype(out_dtype(arr))


def dwt2d_inverse(coeffs, kind) -> np.ndarray:
    """wavelet.py:158-164: columns, then rows."""
    arr = np.asarray(coeffs)
    k = kind_name(kind)
    cols = synthesis_last(np.ascontiguousarray(arr.astype(np.float64).T), k).T
    full = synthesis_last(np.ascontiguousarray(cols), k)
    return np.ascontiguousarray(full).astype(out_dtype(arr))


def fuse_dwt(pan, band, kind) -> np.ndarray:
    """fusion.py:128-150: forward, LL <- band * gain, inverse, cast to the
    PAN dtype. (Validation is the product's job; the oracle assumes valid
    shapes.)"""
    p = np.asarray(pan)
    k = kind_name(kind)
    h, w = p.shape
    coeffs = dwt2d_forward(p.astype(np.float64), k)
    coeffs[: h // 2, : w // 2] = np.asarray(band).astype(np.float64) * _GAIN[k]
    return dwt2d_inverse(coeffs, k).astype(out_dtype(p))


def resample_bilinear(plane, out_w: int, out_h: int) -> np.ndarray:
    """fusion.py:50-81: pixel-centre bilinear with edge clamp."""
    p = np.asarray(plane)
    in_h, in_w = p.shape
    odt = out_dtype(p)
    if (out_w, out_h) == (in_w, in_h):
        return p.astype(odt)
    src = p.astype(np.float64)

    def axis(n_out, n_in):
        s = np.clip((np.arange(n_out) + 0.5) * (n_in / n_out) - 0.5, 0.0, n_in - 1.0)
        i0 = np.floor(s).astype(np.intp)
        return i0, np.minimum(i0 + 1, n_in - 1), s - i0

    x0, x1, fx = axis(out_w, in_w)
    y0, y1, fy = axis(out_h, in_h)
    fy = fy[:, None]
    top, bot = src[y0], src[y1]
    rt = top[:, x0] * (1.0 - fx) + top[:, x1] * fx
    rb = bot[:, x0] * (1.0 - fx) + bot[:, x1] * fx
    return (rt * (1.0 - fy) + rb * fy).astype(odt)


def fuse(pan, bands, kind) -> list[np.ndarray]:
    """fusion.py:170-182 for DwtReplace: resample to half size if needed, then
    one fuse_dwt per band."""
    p = np.asarray(pan)
    h, w = p.shape
    out = []
    for b in bands:
        b = np.asarray(b)
        if b.shape != (h // 2, w // 2):
            b = resample_bilinear(b, w // 2, h // 2)
        out.append(fuse_dwt(p, b, kind))
    return out


# ---------------------------------------------------------------------------
# Windowed oracle: D4 output rows {2i, 2i+1} depend on PAN rows
# 2i-2..2i+3 and MS rows i-1, i (columns likewise) with global periodic wrap.
# Extracting a window with a 2-px wrapped PAN margin (1 px MS), fusing it as a
# whole image and cropping the margin reproduces the global result exactly,
# so windows of scenes too big for the host (65536^2) can be checked.
# ---------------------------------------------------------------------------
def wrapped_window(plane: np.ndarray, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    h, w = plane.shape
    return plane[np.ix_(np.arange(r0, r1) % h, np.arange(c0, c1) % w)]


def fuse_window(pan_fn, band_fns, kind, r0: int, r1: int, c0: int, c1: int,
                margin: int = 4) -> list[np.ndarray]:
    """Fused output rows [r0, r1) x cols [c0, c1) (all even) of a scene whose
    planes are produced on demand: pan_fn(rows, cols) / band_fn(rows, cols)
    return the values at the given absolute (already wrapped) indices.
    margin must be even and >= 2 (PAN px)."""
    k = kind_name(kind)
    m = 0 if k == HAAR else margin
    rows = np.arange(r0 - m, r1 + m)
    cols = np.arange(c0 - m, c1 + m)
    pan = pan_fn(rows, cols)
    mrows = np.arange((r0 - m) // 2, (r1 + m) // 2)
    mcols = np.arange((c0 - m) // 2, (c1 + m) // 2)
    out = []
    for bf in band_fns:
        band = bf(mrows, mcols)
        full = fuse_dwt(pan, band, k)
        out.append(full[m : m + (r1 - r0), m : m + (c1 - c0)])
    return out


def fuse_parallel(pan, bands, kind, threads: int | None = None,
                  strip_rows: int = 512) -> list[np.ndarray]:
    """Exact multi-threaded CPU fusion: row strips with a wrapped 4-row halo
    (numpy releases the GIL), results identical to fuse(). Used as the timed
    CPU baseline (the reference's own fastest CPU path is its thread pool,
    tiling.py:185-189, but that wraps D4 per tile and is not exact)."""
    p = np.asarray(pan)
    h, w = p.shape
    k = kind_name(kind)
    threads = threads or os.cpu_count() or 1
    outs = [np.empty((h, w), dtype=out_dtype(p)) for _ in bands]
    m = 0 if k == HAAR else 4
    starts = list(range(0, h, strip_rows))

    def work(r0):
        r1 = min(h, r0 + strip_rows)
        ridx = np.arange(r0 - m, r1 + m) % h
        sub = p[ridx]
        hh = h // 2
        midx = np.arange((r0 - m) // 2, (r1 + m) // 2) % hh
        for o, b in zip(outs, bands):
            full = fuse_dwt(sub, np.asarray(b)[midx], k)
            o[r0:r1] = full[m : m + (r1 - r0)]

    if h % strip_rows and k == DAUB4 and (h % strip_rows) < 2:
        raise ValueError("strip remainder too small")
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, starts))
    return outs


# ---------------------------------------------------------------------------
# 8 bpp transfer representation
# ---------------------------------------------------------------------------
def quantize(plane) -> np.ndarray:
    """imageio.py:115-123: clamp to [0, 255], then floor(x + 0.5) (half away
    from zero for the clamped, non-negative values), in the plane's dtype."""
    p = np.asarray(plane)
    c = np.minimum(np.maximum(p, p.dtype.type(0.0)), p.dtype.type(255.0))
    return np.floor(c + p.dtype.type(0.5)).astype(np.uint8)


def fuse_tile_quantized(pan_u8, ms_u8, kind) -> list[np.ndarray]:
    """tiling.py:163-172: uint8 tile -> float32 planes -> fuse."""
    return fuse(np.asarray(pan_u8).astype(np.float32),
                [np.asarray(b).astype(np.float32) for b in ms_u8], kind)


def fuse_quantized(pan_u8, ms_u8, kind) -> list[np.ndarray]:
    """tiling.py:268-269: what a worker returns for one 8 bpp tile."""
    return [quantize(p) for p in fuse_tile_quantized(pan_u8, ms_u8, kind)]
