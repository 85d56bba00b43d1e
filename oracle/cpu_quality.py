"""ORACLE — test infrastructure only. Never imported by the product package.

CPU (numpy, float64) restatement of the reference's quality metrics
(/root/reference/pkg/src/wavefuse/metrics.py), used as the checker for the
GPU ERGAS/QNR kernels. Pinned against reference-generated golden vectors in
tests/test_oracle_pinning.py.
"""

from __future__ import annotations

import numpy as np

from .cpu_dwt import resample_bilinear

BLOCK = 32  # metrics.py:17


def degrade(plane, factor: int) -> np.ndarray:
    """metrics.py:31-42: factor x factor block mean."""
    p = np.asarray(plane, dtype=np.float64)
    if factor == 1:
        return p.copy()
    h, w = p.shape
    return p.reshape(h // factor, factor, w // factor, factor).mean(axis=(1, 3))


def blocks(a: np.ndarray) -> np.ndarray:
    """metrics.py:45-54: full 32x32 blocks as (n, 32, 32); partial right and
    bottom blocks are dropped; a plane under 32 in either direction is one
    block."""
    h, w = a.shape
    if h < BLOCK or w < BLOCK:
        return a[None]
    nr, nc = h // BLOCK, w // BLOCK
    t = a[: nr * BLOCK, : nc * BLOCK].reshape(nr, BLOCK, nc, BLOCK)
    return t.transpose(0, 2, 1, 3).reshape(nr * nc, BLOCK, BLOCK)


def q_index(a, b) -> float:
    """metrics.py:57-83: block-averaged universal quality index with
    population moments; den == 0 scores 1 for identical blocks, else 0."""
    ab = blocks(np.asarray(a, dtype=np.float64))
    bb = blocks(np.asarray(b, dtype=np.float64))
    ma = ab.mean(axis=(1, 2))
    mb = bb.mean(axis=(1, 2))
    va = ab.var(axis=(1, 2))
    vb = bb.var(axis=(1, 2))
    cov = ((ab - ma[:, None, None]) * (bb - mb[:, None, None])).mean(axis=(1, 2))
    num = 4.0 * cov * ma * mb
    den = (va + vb) * (ma**2 + mb**2)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = num / den
    bad = den == 0.0
    if bad.any():
        same = np.all(ab[bad] == bb[bad], axis=(1, 2))
        q[bad] = np.where(same, 1.0, 0.0)
    return float(q.mean())


def ergas(fused, ref, ratio: int) -> float:
    """metrics.py:94-119"""
    f = [np.asarray(x, dtype=np.float64) for x in fused]
    r = [np.asarray(x, dtype=np.float64) for x in ref]
    acc = 0.0
    for fb, rb in zip(f, r):
        mu = rb.mean()
        mse = float(np.mean((degrade(fb, ratio) - rb) ** 2))
        acc += mse / (mu * mu)
    return 100.0 / ratio * float(np.sqrt(acc / len(f)))


def upsample(bands, w: int, h: int):
    """metrics.py:122-123"""
    return [b if b.shape == (h, w) else resample_bilinear(b, w, h) for b in bands]


def d_lambda(fused, ms) -> float:
    """metrics.py:126-142"""
    f = [np.asarray(x, dtype=np.float64) for x in fused]
    m = [np.asarray(x, dtype=np.float64) for x in ms]
    n = len(f)
    fh, fw = f[0].shape
    up = upsample(m, fw, fh)
    tot = 0.0
    for k in range(n):
        for l in range(k + 1, n):
            tot += 2.0 * abs(q_index(f[k], f[l]) - q_index(up[k], up[l]))
    return min(1.0, max(0.0, tot / (n * (n - 1))))


def ratio_of(pan_shape, ms_shape) -> int:
    """metrics.py:145-152 (assumes a valid integer ratio)"""
    return pan_shape[0] // ms_shape[0]


def d_s(fused, ms, pan) -> float:
    """metrics.py:155-175"""
    f = [np.asarray(x, dtype=np.float64) for x in fused]
    m = [np.asarray(x, dtype=np.float64) for x in ms]
    p = np.asarray(pan, dtype=np.float64)
    low = degrade(p, ratio_of(p.shape, m[0].shape))
    tot = sum(abs(q_index(fb, p) - q_index(mb, low)) for fb, mb in zip(f, m))
    return min(1.0, max(0.0, tot / len(f)))


def qnr(fused, ms, pan) -> dict:
    """metrics.py:178-199, returned as a dict of the QualityReport fields."""
    f = [np.asarray(x, dtype=np.float64) for x in fused]
    m = [np.asarray(x, dtype=np.float64) for x in ms]
    p = np.asarray(pan, dtype=np.float64)
    ratio = ratio_of(p.shape, m[0].shape)
    fh, fw = f[0].shape
    up = upsample(m, fw, fh)
    per_band = [q_index(fb, ub) for fb, ub in zip(f, up)]
    dl = d_lambda(f, m)
    ds = d_s(f, m, p)
    return {
        "ergas": ergas(f, m, ratio),
        "q_per_band": per_band,
        "d_lambda": dl,
        "d_s": ds,
        "qnr": (1.0 - dl) * (1.0 - ds),
    }
