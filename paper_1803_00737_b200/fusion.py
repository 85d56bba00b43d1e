"""DWT coefficient-replacement fusion, GPU-backed.

Drop-in for the hot path of /root/reference/pkg/src/wavefuse/fusion.py:
`fuse_dwt` (fusion.py:128-150), the `fuse` dispatcher for `DwtReplace`
(fusion.py:153-183), `resample_bilinear` (fusion.py:50-81) and
`method_from_name` (fusion.py:186-196). Same signatures, same validation
order and exception classes (raised before any compute), same dtype rule.

Compute: `fuse` sends all bands of a scene through ONE launch of the fused
kernel (csrc/fuse.cu) that reads PAN once and never materialises the
coefficient image; `fuse_dwt` is the one-band case of the same kernel, so
`fuse(...)[k]` equals `fuse_dwt(pan, ms[k], kind)` bit for bit (the
reference's test_fusion.py:168-187 contract).

numpy inputs go through the library's host-buffer pipeline
(wf_fuse_host_*: H2D, fuse and D2H overlapped in row strips); CUDA tensors
stay on the device (wf_fuse_bands_*).
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .errors import BandCountMismatch, DimensionMismatch, OddDimension, TooSmall
from .wavelet import KIND_CODE, MIN_LEN, WaveletKind

# Default of the `exact` keyword of fuse / fuse_dwt / fuse_tiled. The
# reference's own signatures have no such keyword, so a caller who binds this
# package in place of the reference selects bit-identical
# results with WF_EXACT=1 or set_exact_default(True) instead.
_EXACT_DEFAULT = os.environ.get("WF_EXACT", "0") == "1"


def set_exact_default(flag: bool) -> None:
    """Make exact=True (the reference's float64 operation sequence,
    bit-identical results) the default of fuse / fuse_dwt / fuse_tiled."""
    global _EXACT_DEFAULT
    _EXACT_DEFAULT = bool(flag)


def _exact(flag) -> bool:
    return _EXACT_DEFAULT if flag is None else bool(flag)


# dtypes whose every value a float32 holds exactly: a band of one of these
# enters the reference's LL replacement (fusion.py:149, band * gain in the
# band's own precision) unchanged when cast to a float32 PAN's dtype
_F32_EXACT = {np.dtype(t) for t in (np.float32, np.float16, np.uint8, np.int8, np.uint16,
                                    np.int16, np.bool_)}
_F32_EXACT_T = {torch.float32, torch.float16, torch.bfloat16, torch.uint8, torch.int8,
                torch.int16, torch.bool}


def _f32_exact(b) -> bool:
    if _is_tensor(b):
        return b.dtype in _F32_EXACT_T
    return np.asarray(b).dtype in _F32_EXACT


def _exact_dt(out_dt, bands):
    """Compute dtype of the exact kernels: the PAN's, except that a float32
    PAN with a band float32 cannot hold (float64, wide integers) runs the
    float64 kernels on a float64 copy of the PAN -- the reference keeps such
    a band's full precision in the LL quadrant (fusion.py:148-150) and casts
    only the result to float32, and so does the caller of this (one final
    rounding, the same as astype(float32))."""
    if out_dt == np.float32 and not all(_f32_exact(b) for b in bands):
        return np.float64
    return out_dt


@dataclass(frozen=True)
class DwtReplace:
    """fusion.py:35-40: swap the approximation quadrant of the PAN transform
    for the band data, then invert."""

    kind: WaveletKind


FusionMethod = DwtReplace

# fusion.py:125: Haar (averaging form) has unit DC gain, orthonormal D4 gain 2.
LL_GAIN = {WaveletKind.HAAR: 1.0, WaveletKind.DAUB4: 2.0}


def _shape(x):
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def _is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


# ---------------------------------------------------------------------------
# resample_bilinear (fusion.py:50-81)
# ---------------------------------------------------------------------------
def resample_bilinear(plane, out_w: int, out_h: int):
    """Pixel-centre bilinear resampling, clamped to the source extent.
    Unchanged dimensions return a fresh copy (fusion.py:64-65)."""
    if not _is_tensor(plane):
        plane = np.asarray(plane)
    shape = _shape(plane)
    if len(shape) != 2:
        raise ValueError(f"expected a 2D array, got shape {shape}")
    if out_w < 1 or out_h < 1:
        raise ValueError(f"output size {out_w}x{out_h} must be positive")
    in_h, in_w = shape
    dt = _device.np_out_dtype(plane)
    if (out_w, out_h) == (in_w, in_h):
        if _is_tensor(plane):
            return plane.to(_device.torch_dtype(dt)).clone()
        return plane.astype(dt)
    d_in = _device.to_device(plane, dt)
    d_out = torch.empty((out_h, out_w), dtype=d_in.dtype, device=d_in.device)
    lib = _native.load()
    fn = lib.wf_resample_bilinear_f32 if dt == np.float32 else lib.wf_resample_bilinear_f64
    _native.check(fn(d_in.data_ptr(), in_w, in_h, in_w, d_out.data_ptr(), out_w, out_h, out_w,
                     _device.stream_ptr()))
    return d_out if _is_tensor(plane) else _device.to_host(d_out)


# ---------------------------------------------------------------------------
# fused path
# ---------------------------------------------------------------------------
def _validate_pair(pan_shape, band_shape) -> tuple[int, int]:
    """fusion.py:137-147, then dwt2d_forward's _check_2d (wavelet.py:121-128)."""
    if len(pan_shape) != 2 or len(band_shape) != 2:
        raise ValueError("expected 2D arrays")
    h, w = pan_shape
    if h % 2 or w % 2:
        raise OddDimension(f"panchromatic plane {w}x{h} has an odd dimension")
    if tuple(band_shape) != (h // 2, w // 2):
        raise DimensionMismatch(
            f"band is {band_shape[1]}x{band_shape[0]}, need {w // 2}x{h // 2}"
        )
    return h, w


def _check_min(h: int, w: int, kind: WaveletKind) -> None:
    if h < MIN_LEN[kind] or w < MIN_LEN[kind]:
        raise TooSmall(f"{w}x{h} below minimum {MIN_LEN[kind]} per side")


def _fuse_device(pan_t: torch.Tensor, bands_t: list[torch.Tensor], kind: WaveletKind,
                 out_dt) -> list[torch.Tensor]:
    """All bands in one library call on device-resident tensors."""
    h, w = pan_t.shape
    outs = [torch.empty((h, w), dtype=pan_t.dtype, device=pan_t.device) for _ in bands_t]
    lib = _native.load()
    fn = lib.wf_fuse_bands_f32 if out_dt == np.float32 else lib.wf_fuse_bands_f64
    ms_ptrs = _native.ptr_array([b.data_ptr() for b in bands_t])
    out_ptrs = _native.ptr_array([o.data_ptr() for o in outs])
    _native.check(fn(KIND_CODE[kind], pan_t.data_ptr(), w, ms_ptrs, w // 2, out_ptrs, w,
                     len(bands_t), h, w, _device.stream_ptr()))
    return outs


def _host_out(shape, dt) -> np.ndarray:
    """A fresh numpy output. WF_PINNED_OUT=1: backed by page-locked memory from
    torch's caching host allocator (the D2H lands in it directly, no staging
    copy; the block returns to the cache when the array is freed)."""
    if os.environ.get("WF_PINNED_OUT") == "1":
        tdt = torch.float32 if np.dtype(dt) == np.float32 else torch.float64
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dt)


def _fuse_host(pan: np.ndarray, bands: list[np.ndarray], kind: WaveletKind,
               out_dt, exact: bool = False) -> list[np.ndarray]:
    """All bands through the library's host-buffer pipeline (H2D / fuse / D2H
    overlapped per row strip). exact=True: the strips run the reference-exact
    one-pass kernels with their neighbours' halo rows (wf_ctx_set_exact)."""
    h, w = pan.shape
    pan_c = np.ascontiguousarray(pan, dtype=out_dt)
    band_c = [np.ascontiguousarray(b, dtype=out_dt) for b in bands]
    outs = [_host_out((h, w), out_dt) for _ in bands]
    lib = _native.load()
    fn = lib.wf_fuse_host_f32 if out_dt == np.float32 else lib.wf_fuse_host_f64
    ms_ptrs = _native.ptr_array([b.ctypes.data for b in band_c])
    out_ptrs = _native.ptr_array([o.ctypes.data for o in outs])
    with _device.host_ctx() as ctx:
        _native.check(lib.wf_ctx_set_exact(ctx, 1 if exact else 0))
        _native.check(fn(ctx, KIND_CODE[kind], pan_c.ctypes.data, ms_ptrs, out_ptrs,
                         len(bands), h, w))
    return outs


def _fuse_exact_device(pan_t: torch.Tensor, bands_t: list[torch.Tensor], kind: WaveletKind,
                       out_dt) -> list[torch.Tensor]:
    """Reference-exact path (wf_fuse_dwt_exact_*): float64 forward transform in
    the reference's operation order, LL <- band * gain, float64 inverse, one
    cast -- bit-identical to fusion.py:148-150."""
    h, w = pan_t.shape
    lib = _native.load()
    # the workspace is only used by the WF_EXACT_TRANSFORMS=1 kernel sequence
    ws = torch.empty((h, w) if os.environ.get("WF_EXACT_TRANSFORMS") else (1,),
                     dtype=torch.float64, device=pan_t.device)
    outs = [torch.empty((h, w), dtype=pan_t.dtype, device=pan_t.device) for _ in bands_t]
    if len(bands_t) == 1:  # fuse_dwt: the per-band entry point
        fn = lib.wf_fuse_dwt_exact_f32 if out_dt == np.float32 else lib.wf_fuse_dwt_exact_f64
        _native.check(fn(KIND_CODE[kind], pan_t.data_ptr(), w, bands_t[0].data_ptr(), w // 2,
                         outs[0].data_ptr(), w, h, w, ws.data_ptr(), _device.stream_ptr()))
        return outs
    # fuse: the PAN's forward transform once for every band
    fn = lib.wf_fuse_bands_exact_f32 if out_dt == np.float32 else lib.wf_fuse_bands_exact_f64
    ms_ptrs = _native.ptr_array([b.data_ptr() for b in bands_t])
    out_ptrs = _native.ptr_array([o.data_ptr() for o in outs])
    _native.check(fn(KIND_CODE[kind], pan_t.data_ptr(), w, ms_ptrs, w // 2, out_ptrs, w,
                     len(bands_t), h, w, ws.data_ptr(), _device.stream_ptr()))
    return outs


def fuse_dwt(pan, ms_band, kind: WaveletKind, *, exact: bool | None = None):
    """fusion.py:128-150: transform PAN, overwrite LL with band * gain,
    invert. The band must be exactly half the PAN size per axis. Output dtype
    follows the PAN (float32 iff PAN is float32). exact=True runs the
    reference's own float64 sequence (bit-identical results; one pass,
    1.0-1.4x the fast kernel's time). exact=None: the module default
    (set_exact_default / WF_EXACT)."""
    exact = _exact(exact)
    if not _is_tensor(pan):
        pan = np.asarray(pan)
    if not _is_tensor(ms_band):
        ms_band = np.asarray(ms_band)
    h, w = _validate_pair(_shape(pan), _shape(ms_band))
    _check_min(h, w, kind)
    out_dt = _device.np_out_dtype(pan)
    if exact:
        cdt = _exact_dt(out_dt, [ms_band])
        if _is_tensor(pan):
            out = _fuse_exact_device(_device.to_device(pan, cdt),
                                     [_device.to_device(ms_band, cdt)], kind, cdt)[0]
            return out if cdt == out_dt else out.to(_device.torch_dtype(out_dt))
        out = _fuse_host(pan, [np.asarray(ms_band)], kind, cdt, exact=True)[0]
        return out if cdt == out_dt else out.astype(out_dt)
    if _is_tensor(pan):
        pan_t = _device.to_device(pan, out_dt)
        return _fuse_device(pan_t, [_device.to_device(ms_band, out_dt)], kind, out_dt)[0]
    return _fuse_host(pan, [np.asarray(ms_band)], kind, out_dt)[0]


def fuse(pan, ms, method: FusionMethod, *, exact: bool | None = None):
    """fusion.py:153-183 for DwtReplace: validate the band list, resample
    bands that are not already half-size (bilinear, on the GPU), then fuse
    every band. One launch reads PAN once for up to 8 bands. exact=True: the
    reference's own float64 sequence per band (bit-identical; bands are
    taken in the PAN's dtype). exact=None: the module default
    (set_exact_default / WF_EXACT)."""
    exact = _exact(exact)
    if not _is_tensor(pan):
        pan = np.asarray(pan)
    bands = [b if _is_tensor(b) else np.asarray(b) for b in ms]
    if not bands:
        raise BandCountMismatch("need at least one band")
    first = _shape(bands[0])
    for b in bands[1:]:
        if _shape(b) != first:
            raise DimensionMismatch(f"band sizes differ: {_shape(b)} vs {first}")
    if not isinstance(method, DwtReplace):
        # WA / IHS are outside the north-star path
        raise TypeError(f"unknown fusion method {method!r}")
    shape = _shape(pan)
    if len(shape) != 2:
        raise ValueError("expected 2D arrays")
    h, w = shape
    if h % 2 or w % 2:
        raise OddDimension(f"panchromatic plane {w}x{h} has an odd dimension")
    half = (h // 2, w // 2)
    resampled = [b if _shape(b) == half else resample_bilinear(b, half[1], half[0])
                 for b in bands]
    for b in resampled:
        _validate_pair(shape, _shape(b))
    _check_min(h, w, method.kind)
    out_dt = _device.np_out_dtype(pan)
    if exact:
        cdt = _exact_dt(out_dt, resampled)
        cast = (lambda o: o) if cdt == out_dt else (
            lambda o: o.to(_device.torch_dtype(out_dt)) if _is_tensor(o) else o.astype(out_dt))
        if _is_tensor(pan) or any(_is_tensor(b) for b in resampled):
            outs = _fuse_exact_device(_device.to_device(pan, cdt),
                                      [_device.to_device(b, cdt) for b in resampled],
                                      method.kind, cdt)
            outs = [cast(o) for o in outs]
            return outs if _is_tensor(pan) else [_device.to_host(o) for o in outs]
        # host buffers: the strip pipeline with the exact kernels
        return [cast(o) for o in _fuse_host(pan, [np.asarray(b) for b in resampled],
                                            method.kind, cdt, exact=True)]
    if _is_tensor(pan) or any(_is_tensor(b) for b in resampled):
        pan_t = _device.to_device(pan, out_dt)
        bands_t = [_device.to_device(b, out_dt) for b in resampled]
        outs = _fuse_device(pan_t, bands_t, method.kind, out_dt)
        return outs if _is_tensor(pan) else [_device.to_host(o) for o in outs]
    return _fuse_host(pan, resampled, method.kind, out_dt)


# ---------------------------------------------------------------------------
# 8 bpp transfer representation (tiling.py:155-172,268-269)
# ---------------------------------------------------------------------------
def _u8_to_f32_dev(t: torch.Tensor) -> torch.Tensor:
    h, w = t.shape
    out = torch.empty((h, w), dtype=torch.float32, device=t.device)
    _native.check(_native.load().wf_u8_to_f32(t.data_ptr(), t.stride(0), h, w, out.data_ptr(),
                                              w, _device.stream_ptr()))
    return out


def _quantize_dev(t: torch.Tensor) -> torch.Tensor:
    h, w = t.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=t.device)
    lib = _native.load()
    fn = lib.wf_quantize_f32 if t.dtype == torch.float32 else lib.wf_quantize_f64
    _native.check(fn(t.data_ptr(), t.stride(0), h, w, out.data_ptr(), w, _device.stream_ptr()))
    return out


def quantize(plane):
    """imageio.py:115-123: clamp to [0, 255], then floor(x + 0.5), as uint8 --
    in float32 for float32 planes and float64 otherwise, like numpy."""
    is_t = _is_tensor(plane)
    t = _device.to_device(plane, _device.np_out_dtype(plane))
    shape = tuple(t.shape)
    if t.dim() != 2:  # any shape: quantize is elementwise
        t = t.reshape(1, -1)
    out = _quantize_dev(t).reshape(shape)
    return out if is_t else _device.to_host(out)


def _u8_device(x) -> torch.Tensor:
    dev = _device.require_cuda()
    if _is_tensor(x):
        return (x if x.is_cuda else x.to(dev)).to(torch.uint8).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.uint8)).to(dev)


def fuse_tile_quantized(pan_u8, ms_u8, method: FusionMethod, *, exact: bool | None = None):
    """tiling.py:163-172: fuse one self-contained 8 bpp tile in float32 (the
    worker's computation, cluster.py:297-299); returns float32 planes.
    exact=True: the reference's float64 sequence, so the planes (and their
    quantisation) are the reference worker's bits."""
    pan_f = _u8_to_f32_dev(_u8_device(pan_u8))
    ms_f = [_u8_to_f32_dev(_u8_device(b)) for b in ms_u8]
    out = fuse(pan_f, ms_f, method, exact=exact)
    return out if _is_tensor(pan_u8) else [_device.to_host(o) for o in out]


def fuse_quantized(pan_u8, ms_u8, method: FusionMethod, *, exact: bool | None = None):
    """[quantize(p) for p in fuse_tile_quantized(pan_u8, ms_u8, method)]
    (tiling.py:268-269) in ONE pass: uint8 PAN/MS in, uint8 out, the quantize
    fused into the store (1 + 1.25 B per PAN px per band instead of 9), and
    byte-identical to the reference worker in every mode: Haar is exact in
    integer lanes; D4 computes in float32 with a proven error bound and
    recomputes in float64 the 0.4% of pixels that lie near a rounding
    boundary (csrc/fuse_tma.cu, v3). Shapes the 8 bpp kernels do not cover (MS
    not half size, W % 16 / 32) take the reference-exact float64 kernels plus
    the GPU quantize, which are byte-identical too. exact=True (D4) takes that
    reference-order route for every pixel."""
    exact = _exact(exact)
    if not isinstance(method, DwtReplace):
        raise TypeError(f"unknown fusion method {method!r}")
    is_t = _is_tensor(pan_u8)
    pan_shape = _shape(pan_u8)
    bands = list(ms_u8)
    if not bands:
        raise BandCountMismatch("need at least one band")
    h, w = pan_shape
    if h % 2 or w % 2:
        raise OddDimension(f"panchromatic plane {w}x{h} has an odd dimension")
    half = (h // 2, w // 2)
    fast = all(_shape(b) == half for b in bands) and (
        w % 16 == 0 if method.kind is WaveletKind.HAAR else w % 32 == 0) and not (
        exact and method.kind is WaveletKind.DAUB4)
    if fast:
        _check_min(h, w, method.kind)
        lib = _native.load()
        code = KIND_CODE[method.kind]
        if is_t:
            pan_t = _u8_device(pan_u8)
            bands_t = [_u8_device(b) for b in bands]
            outs = [torch.empty((h, w), dtype=torch.uint8, device=pan_t.device) for _ in bands]
            _native.check(lib.wf_fuse_bands_u8(
                code, pan_t.data_ptr(), w, _native.ptr_array([b.data_ptr() for b in bands_t]),
                w // 2, _native.ptr_array([o.data_ptr() for o in outs]), w, len(bands), h, w,
                _device.stream_ptr()))
            return outs
        pan_c = np.ascontiguousarray(np.asarray(pan_u8), dtype=np.uint8)
        band_c = [np.ascontiguousarray(np.asarray(b), dtype=np.uint8) for b in bands]
        outs = [np.empty((h, w), dtype=np.uint8) for _ in bands]
        with _device.host_ctx() as ctx:
            _native.check(lib.wf_fuse_host_u8(
                ctx, code, pan_c.ctypes.data, _native.ptr_array([b.ctypes.data for b in band_c]),
                _native.ptr_array([o.ctypes.data for o in outs]), len(bands), h, w))
        return outs
    # bytes out: the reference-exact kernels, so the quantised bytes are the
    # reference's whatever `exact` says
    fused = fuse_tile_quantized(_u8_device(pan_u8), [_u8_device(b) for b in bands], method,
                                exact=True)
    outs = [_quantize_dev(f) for f in fused]
    return outs if is_t else [_device.to_host(o) for o in outs]


def method_from_name(name: str, weight: float = 0.5) -> FusionMethod:
    """fusion.py:186-196 (the DWT names; wa/ihs are out of scope here)."""
    if name == "hdwt":
        return DwtReplace(WaveletKind.HAAR)
    if name == "ddwt":
        return DwtReplace(WaveletKind.DAUB4)
    raise ValueError(f"unknown method name {name!r}")
