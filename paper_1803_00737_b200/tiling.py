"""Tiled fusion with the reference's per-tile semantics, on the GPU
(SURVEY.md 8(f) row f4).

Drop-in for the DWT part of /root/reference/pkg/src/wavefuse/tiling.py:
`TileGrid`, `plan_grid` (tiling.py:38-86) and `fuse_tiled` (tiling.py:213-273)
with `workers` and `transfer_8bpp`. Every tile is fused as its own image --
periodic wrap INSIDE the tile, the reference's documented choice "rather than
add halo exchange" (tiling.py:1-12) -- by launching the fused
kernel on a strided window of the device-resident scene (pitch = scene width),
so no tile is ever copied. (For exact whole-scene results across GPUs use
strips.py, which exchanges halos instead.)
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .errors import (BandCountMismatch, DimensionMismatch, MissingTile, NotDivisible, OddTile,
                     TooSmall)
from .fusion import (
    DwtReplace,
    FusionMethod,
    _exact,
    _exact_dt,
    _quantize_dev,
    _u8_device,
    _u8_to_f32_dev,
    resample_bilinear,
)
from .wavelet import KIND_CODE, MIN_LEN, WaveletKind


@dataclass(frozen=True)
class TileGrid:
    """tiling.py:38-58: equal-parts partition, sizes in pixels."""

    grid_w: int
    grid_h: int
    pan_tile_w: int
    pan_tile_h: int
    ms_tile_w: int
    ms_tile_h: int

    @property
    def tile_count(self) -> int:
        return self.grid_w * self.grid_h

    @property
    def pan_w(self) -> int:
        return self.grid_w * self.pan_tile_w

    @property
    def pan_h(self) -> int:
        return self.grid_h * self.pan_tile_h


def plan_grid(pan_w: int, pan_h: int, grid_w: int, grid_h: int) -> TileGrid:
    """tiling.py:72-86"""
    if grid_w < 1 or grid_h < 1:
        raise ValueError(f"grid {grid_w}x{grid_h} must be at least 1x1")
    if pan_w % grid_w or pan_h % grid_h:
        raise NotDivisible(f"{pan_w}x{pan_h} not divisible into {grid_w}x{grid_h} tiles")
    tile_w, tile_h = pan_w // grid_w, pan_h // grid_h
    if tile_w % 2 or tile_h % 2:
        raise OddTile(f"tile {tile_w}x{tile_h} has an odd dimension")
    return TileGrid(grid_w, grid_h, tile_w, tile_h, tile_w // 2, tile_h // 2)


@dataclass(frozen=True)
class Tile:
    """tiling.py Tile: grid position (row, col), the PAN crop and the
    half-resolution band crops."""

    index: tuple
    pan: object
    ms: list


def _crop(plane, row: int, col: int, tile_w: int, tile_h: int):
    """One tile of a plane as a fresh contiguous array: a device copy for a
    CUDA tensor (the plane never leaves HBM), a host copy for numpy."""
    piece = plane[row * tile_h:(row + 1) * tile_h, col * tile_w:(col + 1) * tile_w]
    if isinstance(piece, torch.Tensor):
        return piece.contiguous() if not piece.is_contiguous() else piece.clone()
    return np.ascontiguousarray(piece)


def split(pan, ms, grid: TileGrid) -> list:
    """tiling.py:93-118: cut the PAN and half-resolution bands into row-major
    contiguous tiles. Pure data movement (no arithmetic): CUDA tensors are
    cropped on the device, numpy planes on the host, as the reference does.
    (The fused paths never call this: fuse_tiled launches the kernels on
    strided windows of the whole plane instead of copying tiles.)"""
    pan_arr = pan if isinstance(pan, torch.Tensor) else np.asarray(pan)
    bands = [b if isinstance(b, torch.Tensor) else np.asarray(b) for b in ms]
    if _shape(pan_arr) != (grid.pan_h, grid.pan_w):
        raise DimensionMismatch(
            f"panchromatic {_shape(pan_arr)} does not match grid {grid.pan_w}x{grid.pan_h}")
    half = (grid.pan_h // 2, grid.pan_w // 2)
    for b in bands:
        if _shape(b) != half:
            raise DimensionMismatch(f"band {_shape(b)} is not half-size {half}")
    tiles = []
    for row in range(grid.grid_h):
        for col in range(grid.grid_w):
            tiles.append(Tile((row, col),
                              _crop(pan_arr, row, col, grid.pan_tile_w, grid.pan_tile_h),
                              [_crop(b, row, col, grid.ms_tile_w, grid.ms_tile_h)
                               for b in bands]))
    return tiles


def merge(tiles, grid: TileGrid) -> list:
    """tiling.py:121-152: assemble per-tile fused bands (row-major order)
    into full planes, placed by list index, never by arrival order. Device
    tiles are assembled in HBM (tensor out), host tiles on the host."""
    tiles = list(tiles)
    if len(tiles) != grid.tile_count:
        raise MissingTile(f"got {len(tiles)} tiles, grid has {grid.tile_count}")
    for i, t in enumerate(tiles):
        if t is None:
            raise MissingTile(f"tile index {i} is absent")
    first = tiles[0]
    band_count = len(first)
    th, tw = grid.pan_tile_h, grid.pan_tile_w
    for t in tiles:
        if len(t) != band_count:
            raise DimensionMismatch(f"band counts differ: {len(t)} vs {band_count}")
        for b in t:
            if _shape(b) != (th, tw):
                raise DimensionMismatch(f"tile band {_shape(b)} is not {tw}x{th}")
    on_dev = isinstance(first[0], torch.Tensor)
    if on_dev:
        out = [torch.empty((grid.pan_h, grid.pan_w), dtype=first[k].dtype,
                           device=first[k].device) for k in range(band_count)]
    else:
        out = [np.empty((grid.pan_h, grid.pan_w), dtype=np.asarray(first[k]).dtype)
               for k in range(band_count)]
    for i, t in enumerate(tiles):
        row, col = divmod(i, grid.grid_w)
        for k in range(band_count):
            src = t[k]
            if on_dev and not isinstance(src, torch.Tensor):
                src = torch.as_tensor(np.asarray(src), device=out[k].device)
            out[k][row * th:(row + 1) * th, col * tw:(col + 1) * tw] = src
    return out


def padded_dims(w: int, h: int, grid_w: int, grid_h: int) -> tuple[int, int]:
    """tiling.py:276-285"""
    if grid_w < 1 or grid_h < 1:
        raise ValueError(f"grid {grid_w}x{grid_h} must be at least 1x1")
    step_w, step_h = 2 * grid_w, 2 * grid_h
    return (w + step_w - 1) // step_w * step_w, (h + step_h - 1) // step_h * step_h


def _shape(x):
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def pad_edge(plane, out_w: int, out_h: int):
    """tiling.py:285-293: grow a plane to out_w x out_h by replicating its last
    row and column (np.pad mode="edge"); always a fresh array. One launch of
    wf_pad_edge_* on the GPU; numpy in -> numpy out, tensor in -> tensor out."""
    is_t = isinstance(plane, torch.Tensor)
    if not is_t:
        plane = np.asarray(plane)
    h, w = _shape(plane)
    if out_w < w or out_h < h:
        raise ValueError(f"cannot pad {w}x{h} down to {out_w}x{out_h}")
    dt = _device.np_out_dtype(plane)
    src = _device.to_device(plane, dt)
    if (out_w, out_h) == (w, h):
        out = src.clone() if src is plane else src  # always a fresh array (plane.copy())
    else:
        out = torch.empty((out_h, out_w), dtype=src.dtype, device=src.device)
        fn = _native.load().wf_pad_edge_f32 if dt == np.float32 else _native.load().wf_pad_edge_f64
        _native.check(fn(src.data_ptr(), src.stride(0), h, w, out.data_ptr(), out_w, out_h, out_w,
                         _device.stream_ptr()))
    return out if is_t else _device.to_host(out)


def pad_inputs(pan, ms, grid_w: int, grid_h: int):
    """tiling.py:296-310: edge-pad the PAN to grid-compatible dimensions and
    every band in proportion ((bw * pw + w - 1) // w per axis), so the bands
    keep covering the same region. Returns (pan, list(ms)) unchanged when no
    padding is needed."""
    h, w = _shape(pan)
    pw, ph = padded_dims(w, h, grid_w, grid_h)
    if (pw, ph) == (w, h):
        return pan, list(ms)
    bands = []
    for band in ms:
        bh, bw = _shape(band)
        bands.append(pad_edge(band, (bw * pw + w - 1) // w, (bh * ph + h - 1) // h))
    return pad_edge(pan, pw, ph), bands


def _window_fuse(kind: WaveletKind, pan: torch.Tensor, ms: list[torch.Tensor],
                 out: list[torch.Tensor], grid: TileGrid, exact: bool = False) -> None:
    """One fused launch per tile on strided windows of the device scene; each
    tile wraps periodically within itself. exact=True runs the reference's
    float64 operation order per tile for all bands (wf_fuse_bands_exact_*)."""
    lib = _native.load()
    esz = pan.element_size()
    tw, th = grid.pan_tile_w, grid.pan_tile_h
    pp, mp, op = pan.stride(0), ms[0].stride(0), out[0].stride(0)
    s = _device.stream_ptr()
    code = KIND_CODE[kind]
    if exact:  # one launch per tile for all bands (the one-pass exact kernels)
        fn = (lib.wf_fuse_bands_exact_f32 if pan.dtype == torch.float32
              else lib.wf_fuse_bands_exact_f64)
        ws = torch.empty(1, dtype=torch.float64, device=pan.device)  # unused by the one-pass path
        if os.environ.get("WF_EXACT_TRANSFORMS"):
            ws = torch.empty((th, tw), dtype=torch.float64, device=pan.device)
    else:
        fn = {torch.float32: lib.wf_fuse_bands_f32, torch.float64: lib.wf_fuse_bands_f64,
              torch.uint8: lib.wf_fuse_bands_u8}[pan.dtype]
    for row in range(grid.grid_h):
        for col in range(grid.grid_w):
            r0, c0 = row * th, col * tw
            pan_p = pan.data_ptr() + (r0 * pp + c0) * esz
            ms_a = [m.data_ptr() + ((r0 // 2) * mp + c0 // 2) * esz for m in ms]
            out_a = [o.data_ptr() + (r0 * op + c0) * esz for o in out]
            if exact:
                _native.check(fn(code, pan_p, pp, _native.ptr_array(ms_a), mp,
                                 _native.ptr_array(out_a), op, len(ms), th, tw, ws.data_ptr(), s))
            else:
                _native.check(fn(code, pan_p, pp, _native.ptr_array(ms_a), mp,
                                 _native.ptr_array(out_a), op, len(ms), th, tw, s))


def _u8_windows_ok(grid: TileGrid, kind: WaveletKind) -> bool:
    # the 8 bpp kernels need 16-byte aligned PAN and MS window bases and row
    # pitches: tile widths (hence MS tile widths x2) that are multiples of 32
    return grid.pan_tile_w % 32 == 0 and grid.pan_w % 32 == 0


def fuse_tiled(pan, ms, method: FusionMethod, grid: TileGrid, workers: int = 1,
               transfer_8bpp: bool = False, *, exact: bool | None = None):
    """tiling.py:213-273 for DwtReplace. `workers` is accepted for signature
    compatibility (the GPU fuses tiles, not a thread pool). Plain mode
    resamples bands globally, then fuses every tile with per-tile wrap (float
    output, pan dtype); exact=True fuses each tile in the reference's own
    float64 operation order (bit-identical to the reference). transfer_8bpp
    reproduces the distributed pipeline: inputs quantised to uint8
    (wire_planes, tiling.py:192-210), each tile fused and quantised
    (tiling.py:163-172, 268-269) -- byte-identical to the reference's workers
    (the byte-exact 8 bpp kernels, or the reference-exact float64 kernels
    plus the quantize for tile shapes they do not cover)."""
    exact = _exact(exact)
    if workers < 1:
        raise ValueError(f"workers {workers} must be >= 1")
    is_t = isinstance(pan, torch.Tensor)
    if not is_t:
        pan = np.asarray(pan)
    if _shape(pan) != (grid.pan_h, grid.pan_w):
        raise DimensionMismatch(
            f"panchromatic {_shape(pan)} does not match grid {grid.pan_w}x{grid.pan_h}")
    bands = [b if isinstance(b, torch.Tensor) else np.asarray(b) for b in ms]
    if not bands:
        raise BandCountMismatch("need at least one band")
    for b in bands[1:]:
        if _shape(b) != _shape(bands[0]):
            raise DimensionMismatch(f"band sizes differ: {_shape(b)} vs {_shape(bands[0])}")
    if not isinstance(method, DwtReplace):
        raise TypeError(f"unknown fusion method {method!r}")
    kind = method.kind
    th, tw = grid.pan_tile_h, grid.pan_tile_w
    if th < MIN_LEN[kind] or tw < MIN_LEN[kind]:
        raise TooSmall(f"{tw}x{th} below minimum {MIN_LEN[kind]} per side")
    half = (grid.pan_h // 2, grid.pan_w // 2)

    if transfer_8bpp:
        # wire_planes: bands to half size (bilinear), then everything to uint8
        low = [b if _shape(b) == half else resample_bilinear(b, half[1], half[0]) for b in bands]

        def to_u8(x):  # uint8 passes through; other planes are quantised in their
            # own dtype rule (float32 iff float32, else float64), like the
            # reference's quantize on the numpy plane (imageio.py:115-123)
            is_u8 = x.dtype == (torch.uint8 if isinstance(x, torch.Tensor) else np.uint8)
            return _u8_device(x) if is_u8 else _quantize_dev(
                _device.to_device(x, _device.np_out_dtype(x)))

        pan_u8 = to_u8(pan)
        ms_u8 = [to_u8(b) for b in low]
        if _u8_windows_ok(grid, kind) and not (exact and kind is WaveletKind.DAUB4):
            outs = [torch.empty_like(pan_u8) for _ in ms_u8]
            _window_fuse(kind, pan_u8, ms_u8, outs, grid)
        else:  # the reference's float64 kernels + quantize: the worker's bytes
            pan_f = _u8_to_f32_dev(pan_u8)
            ms_f = [_u8_to_f32_dev(b) for b in ms_u8]
            fo = [torch.empty_like(pan_f) for _ in ms_f]
            _window_fuse(kind, pan_f, ms_f, fo, grid, exact=True)
            outs = [_quantize_dev(f) for f in fo]
        return outs if is_t else [_device.to_host(o) for o in outs]

    out_dt = _device.np_out_dtype(pan)
    sized = [b if _shape(b) == half else resample_bilinear(b, half[1], half[0]) for b in bands]
    # exact: a float32 PAN with float64 bands runs the float64 kernels and
    # casts once at the end, like the reference (fusion._exact_dt)
    dt = _exact_dt(out_dt, sized) if exact else out_dt
    pan_t = _device.to_device(pan, dt)
    ms_t = [_device.to_device(b, dt) for b in sized]
    outs = [torch.empty_like(pan_t) for _ in ms_t]
    _window_fuse(kind, pan_t, ms_t, outs, grid, exact=exact)
    if dt != out_dt:
        outs = [o.to(_device.torch_dtype(out_dt)) for o in outs]
    return outs if is_t else [_device.to_host(o) for o in outs]

