"""PNM front end of the fusion path.

Drop-in for /root/reference/pkg/src/wavefuse/imageio.py (read_pnm,
write_pnm, to_plane, quantize) plus the data path of the reference CLI's
`fuse` command (cli.py:113-165) as one call, `fuse_pnm`.

Split of the work:
- PGM/PPM headers are a few bytes of sequential text: parsed and written on
  the host, with the reference's rules and exception classes.
- Everything per pixel runs on the GPU (csrc/raster.cu): channel extraction
  and uint8 -> float conversion fused with edge padding
  (wf_raster_to_plane_*), the fusion itself, and crop + quantize + channel
  interleave of the result (wf_planes_to_raster_*). A scene therefore
  crosses PCIe as 8-bit rasters: 1 byte per pixel and channel each way,
  instead of 4-byte float planes.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _native
from .errors import ChannelOutOfRange, MalformedHeader, Truncated, UnsupportedFormat
from .fusion import FusionMethod, quantize
from .tiling import fuse_tiled, padded_dims, plan_grid

__all__ = ["read_pnm", "write_pnm", "to_plane", "quantize", "fuse_pnm", "PnmRaster"]

_SPACE = frozenset(b" \t\n\r\x0b\x0c")
_DIGITS = frozenset(b"0123456789")


def _header_ints(data: bytes, pos: int, count: int) -> tuple[list[int], int]:
    """imageio.py:22-43: `count` decimal tokens from `pos`; whitespace runs and
    '#'-to-end-of-line comments may precede each token."""
    out: list[int] = []
    n = len(data)
    while len(out) < count:
        while pos < n and data[pos] in _SPACE:
            pos += 1
        if pos < n and data[pos] == 0x23:  # '#': comment through the newline
            nl = data.find(b"\n", pos)
            if nl < 0:
                raise MalformedHeader("unterminated comment in header")
            pos = nl + 1
            continue
        end = pos
        while end < n and data[end] in _DIGITS:
            end += 1
        if end == pos:
            raise MalformedHeader("expected integer in header")
        out.append(int(data[pos:end]))
        pos = end
    return out, pos


class PnmRaster:
    """A decoded binary PGM/PPM header: dimensions, channel count and where
    the payload starts (maxval is always 255)."""

    __slots__ = ("width", "height", "channels", "offset")

    def __init__(self, width: int, height: int, channels: int, offset: int):
        self.width, self.height, self.channels, self.offset = width, height, channels, offset

    @property
    def nbytes(self) -> int:
        return self.width * self.height * self.channels

    @property
    def shape(self) -> tuple[int, ...]:
        if self.channels == 1:
            return (self.height, self.width)
        return (self.height, self.width, self.channels)

    @classmethod
    def parse(cls, data: bytes) -> "PnmRaster":
        """imageio.py:46-87 up to the payload, with its exception rules."""
        if len(data) < 2:
            raise MalformedHeader("input shorter than a magic number")
        channels = {b"P5": 1, b"P6": 3}.get(bytes(data[:2]))
        if channels is None:
            raise UnsupportedFormat("expected binary PGM (P5) or PPM (P6)")
        if len(data) < 3 or data[2] not in _SPACE:
            raise MalformedHeader("magic number not followed by whitespace")
        (w, h, maxval), pos = _header_ints(data, 2, 3)
        if w <= 0 or h <= 0:
            raise MalformedHeader(f"invalid dimensions {w}x{h}")
        if maxval != 255:
            raise UnsupportedFormat(f"maxval {maxval} not supported, need 255")
        if pos >= len(data) or data[pos] not in _SPACE:  # exactly one byte
            raise MalformedHeader("missing whitespace after maxval")
        r = cls(w, h, channels, pos + 1)
        have = max(0, len(data) - r.offset)
        if have < r.nbytes:
            raise Truncated(f"payload has {have} bytes, header promises {r.nbytes}")
        return r


def read_pnm(data: bytes, *, device: bool = False):
    """imageio.py:46-87: decode a binary PGM (P5) or PPM (P6), maxval 255, to
    uint8 (h, w) or (h, w, 3). device=True returns a CUDA tensor (the payload
    goes host -> HBM as raw bytes)."""
    r = PnmRaster.parse(data)
    payload = np.frombuffer(data, dtype=np.uint8, count=r.nbytes, offset=r.offset)
    if device:
        return torch.from_numpy(payload.copy()).to(_device.require_cuda()).view(*r.shape)
    return payload.reshape(r.shape).copy()


def write_pnm(raster) -> bytes:
    """imageio.py:90-101: encode a uint8 raster, (h, w) -> PGM, (h, w, 3) ->
    PPM. Accepts numpy arrays and CUDA tensors."""
    if isinstance(raster, torch.Tensor):
        if raster.dtype != torch.uint8:
            raise UnsupportedFormat(f"raster dtype must be uint8, got {raster.dtype}")
        r = raster.contiguous().cpu().numpy()
    else:
        r = np.asarray(raster)
        if r.dtype != np.uint8:
            raise UnsupportedFormat(f"raster dtype must be uint8, got {r.dtype}")
    if r.ndim == 2:
        magic = b"P5"
    elif r.ndim == 3 and r.shape[2] == 3:
        magic = b"P6"
    else:
        raise UnsupportedFormat(f"raster shape {r.shape} is not (h, w) or (h, w, 3)")
    return b"%s\n%d %d\n255\n" % (magic, r.shape[1], r.shape[0]) + np.ascontiguousarray(r).tobytes()


def _raster_device(raster) -> torch.Tensor:
    if isinstance(raster, torch.Tensor):
        t = raster if raster.is_cuda else raster.to(_device.require_cuda())
        return t.to(torch.uint8).contiguous()
    arr = np.ascontiguousarray(np.asarray(raster), dtype=np.uint8)
    return torch.from_numpy(arr).to(_device.require_cuda())


def _plane_dev(r: torch.Tensor, channel: int, out_h: int | None = None,
               out_w: int | None = None, dtype=torch.float32) -> torch.Tensor:
    """wf_raster_to_plane_*: channel `channel` of a device raster as a float
    plane, edge-padded to out_h x out_w."""
    h, w = r.shape[:2]
    ch = 1 if r.dim() == 2 else r.shape[2]
    oh, ow = out_h or h, out_w or w
    out = torch.empty((oh, ow), dtype=dtype, device=r.device)
    lib = _native.load()
    fn = lib.wf_raster_to_plane_f32 if dtype == torch.float32 else lib.wf_raster_to_plane_f64
    _native.check(fn(r.data_ptr(), h, w, ch, channel, out.data_ptr(), ow, oh, ow,
                     _device.stream_ptr()))
    return out


def to_plane(raster, channel: int = 0):
    """imageio.py:104-112: one channel as a float32 plane on the 0..255 scale.
    numpy in -> numpy out, tensor in -> tensor out."""
    is_t = isinstance(raster, torch.Tensor)
    shape = tuple(raster.shape) if is_t else np.shape(raster)
    channels = 1 if len(shape) == 2 else shape[2]
    if channel < 0 or channel >= channels:
        raise ChannelOutOfRange(f"channel {channel} of {channels}")
    out = _plane_dev(_raster_device(raster), channel)
    return out if is_t else _device.to_host(out)


def _raster_from_planes(planes: list[torch.Tensor], h: int, w: int) -> np.ndarray:
    """wf_planes_to_raster_*: quantize the top-left h x w of every plane and
    interleave, then one device -> host copy."""
    np_ = len(planes)
    dev = planes[0].device
    raster = torch.empty((h, w, np_) if np_ > 1 else (h, w), dtype=torch.uint8, device=dev)
    lib = _native.load()
    fn = (lib.wf_planes_to_raster_f32 if planes[0].dtype == torch.float32
          else lib.wf_planes_to_raster_f64)
    _native.check(fn(_native.ptr_array([p.data_ptr() for p in planes]), np_, planes[0].stride(0),
                     h, w, raster.data_ptr(), _device.stream_ptr()))
    return _device.to_host(raster)


def fuse_pnm(pan: bytes, ms: list[bytes], method: FusionMethod, grid: tuple[int, int] = (1, 1),
             *, exact: bool | None = None) -> list[bytes]:
    """The data path of the reference's `wavefuse fuse` (cli.py:147-165) for
    DwtReplace methods, in memory: PGM PAN + band files (one PPM = 3 bands,
    else one PGM per band) -> the PNM files it would write (cli.py:135-144):
    one PPM for 3 bands, one PGM for 1 band, else one PGM per band.

    GPU pipeline: raw payloads H2D -> planes with the edge padding of
    pad_inputs fused in (tiling.py:296-310) -> fuse_tiled on `grid` (per-tile
    wrap, tiling.py:213-273) -> crop + quantize + interleave -> D2H.
    Every tile is fused in the reference's float64 operation order by
    default (exact=None -> True here: the outputs are bytes, and they are the
    reference CLI's bytes); exact=False takes the float32 kernels (within
    1e-3 before the quantize, so a byte can differ by one where a value sits
    at a rounding boundary)."""
    pr = PnmRaster.parse(pan)
    if pr.channels != 1:
        raise ValueError("panchromatic image must be grayscale")
    rasters = [PnmRaster.parse(m) for m in ms]
    if not rasters:
        raise ValueError("need at least one band file")
    if len(rasters) > 1 and any(r.channels != 1 for r in rasters):
        raise ValueError("band files must be grayscale")
    h, w = pr.height, pr.width
    gw, gh = grid
    pw, ph = padded_dims(w, h, gw, gh)
    dev = _device.require_cuda()

    def upload(data: bytes, r: PnmRaster) -> torch.Tensor:
        payload = np.frombuffer(data, dtype=np.uint8, count=r.nbytes, offset=r.offset)
        return torch.from_numpy(payload.copy()).to(dev).view(*r.shape)

    pan_t = _plane_dev(upload(pan, pr), 0, ph, pw)
    bands = []
    for data, r in zip(ms, rasters):
        t = upload(data, r)
        # pad_inputs: each band grows in proportion to the PAN (tiling.py:305-309)
        bh = (r.height * ph + h - 1) // h
        bw = (r.width * pw + w - 1) // w
        bands += [_plane_dev(t, c, bh, bw) for c in range(r.channels)]
    fused = fuse_tiled(pan_t, bands, method, plan_grid(pw, ph, gw, gh),
                       exact=True if exact is None else exact)
    if len(fused) == 3:
        return [write_pnm(_raster_from_planes(fused, h, w))]
    return [write_pnm(_raster_from_planes([f], h, w)) for f in fused]
