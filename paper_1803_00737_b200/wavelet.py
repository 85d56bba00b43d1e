"""Single-level Haar / Daubechies-4 transforms, GPU-backed.

Drop-in for /root/reference/pkg/src/wavefuse/wavelet.py: same names, same
signatures, same coefficient layout ([approx | detail] per axis, LL top-left),
same periodic boundary, same dtype rule and same exceptions raised before any
compute. The arithmetic runs in the sm_100a library (transforms.cu) in float64
with the reference's operation order, so results are bit-identical to the
reference for float64 and float32 inputs alike.

Inputs may be numpy arrays (result: numpy) or CUDA torch tensors (result: a
CUDA tensor, no host round trip).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _device, _native
from .errors import OddDimension, OddLength, TooShort, TooSmall


class WaveletKind(Enum):
    """wavelet.py:27-29"""

    HAAR = "haar"
    DAUB4 = "daub4"


KIND_CODE = {WaveletKind.HAAR: _native.HAAR, WaveletKind.DAUB4: _native.DAUB4}


@dataclass(frozen=True)
class FilterBank:
    """wavelet.py:32-45: analysis low/high quads and the interleaved
    synthesis quads for even/odd output samples."""

    analysis_low: np.ndarray
    analysis_high: np.ndarray
    synthesis_even: np.ndarray
    synthesis_odd: np.ndarray


def d4_filters() -> FilterBank:
    """wavelet.py:48-63. A constant table; the device computes the same
    doubles itself (csrc/wf_common.cuh d4_taps)."""
    root3 = math.sqrt(3.0)
    norm = 4.0 * math.sqrt(2.0)
    h = np.array([(1.0 + root3) / norm, (3.0 + root3) / norm,
                  (3.0 - root3) / norm, (1.0 - root3) / norm])
    g = np.array([h[3], -h[2], h[1], -h[0]])
    even = np.array([h[2], g[2], h[0], g[0]])
    odd = np.array([h[3], g[3], h[1], g[1]])
    for a in (h, g, even, odd):
        a.setflags(write=False)
    return FilterBank(h, g, even, odd)


MIN_LEN = {WaveletKind.HAAR: 2, WaveletKind.DAUB4: 4}  # wavelet.py:66


def _shape(x) -> tuple[int, ...]:
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def check_1d(shape, kind: WaveletKind) -> None:
    """wavelet.py:112-118"""
    if len(shape) != 1:
        raise ValueError(f"expected a 1D array, got shape {shape}")
    if shape[0] < MIN_LEN[kind]:
        raise TooShort(f"length {shape[0]} below minimum {MIN_LEN[kind]}")
    if shape[0] % 2:
        raise OddLength(f"length {shape[0]} is odd")


def check_2d(shape, kind: WaveletKind) -> None:
    """wavelet.py:121-128"""
    if len(shape) != 2:
        raise ValueError(f"expected a 2D array, got shape {shape}")
    h, w = shape
    if h < MIN_LEN[kind] or w < MIN_LEN[kind]:
        raise TooSmall(f"{w}x{h} below minimum {MIN_LEN[kind]} per side")
    if h % 2 or w % 2:
        raise OddDimension(f"{w}x{h} has an odd dimension")


def _finish(x, out: torch.Tensor):
    return out if isinstance(x, torch.Tensor) else _device.to_host(out)


def _rows_call(x, kind: WaveletKind, inverse: bool):
    if not isinstance(x, torch.Tensor):
        x = np.asarray(x)
    check_1d(_shape(x), kind)
    dt = _device.np_out_dtype(x)
    d_in = _device.to_device(x, dt).reshape(1, -1)
    d_out = torch.empty_like(d_in)
    n = d_in.shape[1]
    lib = _native.load()
    fn = {
        (False, np.float32): lib.wf_dwt_rows_forward_f32,
        (False, np.float64): lib.wf_dwt_rows_forward_f64,
        (True, np.float32): lib.wf_dwt_rows_inverse_f32,
        (True, np.float64): lib.wf_dwt_rows_inverse_f64,
    }[(inverse, dt)]
    _native.check(fn(KIND_CODE[kind], d_in.data_ptr(), n, d_out.data_ptr(), n, 1, n,
                     _device.stream_ptr()))
    return _finish(x, d_out.reshape(-1))


def dwt1d_forward(x, kind: WaveletKind):
    """wavelet.py:131-139: [approx | detail] of an even-length vector."""
    return _rows_call(x, kind, inverse=False)


def dwt1d_inverse(coeffs, kind: WaveletKind):
    """wavelet.py:142-146"""
    return _rows_call(coeffs, kind, inverse=True)


def _plane_call(x, kind: WaveletKind, inverse: bool):
    if not isinstance(x, torch.Tensor):
        x = np.asarray(x)
    check_2d(_shape(x), kind)
    dt = _device.np_out_dtype(x)
    d_in = _device.to_device(x, dt)
    d_out = torch.empty_like(d_in)
    h, w = d_in.shape
    lib = _native.load()
    fn = {
        (False, np.float32): lib.wf_dwt2d_forward_f32,
        (False, np.float64): lib.wf_dwt2d_forward_f64,
        (True, np.float32): lib.wf_dwt2d_inverse_f32,
        (True, np.float64): lib.wf_dwt2d_inverse_f64,
    }[(inverse, dt)]
    _native.check(fn(KIND_CODE[kind], d_in.data_ptr(), w, d_out.data_ptr(), w, h, w,
                     _device.stream_ptr()))
    return _finish(x, d_out)


def dwt2d_forward(plane, kind: WaveletKind):
    """wavelet.py:149-155: rows then columns; LL top-left, HL top-right,
    LH bottom-left, HH bottom-right."""
    return _plane_call(plane, kind, inverse=False)


def dwt2d_inverse(coeffs, kind: WaveletKind):
    """wavelet.py:158-164: columns then rows."""
    return _plane_call(coeffs, kind, inverse=True)
