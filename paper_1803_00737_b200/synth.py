"""Synthetic Landsat-7-shaped scenes.

Two generators:

* `synth_scene(w, h, bands, seed)` — the reference's own recipe
  (/root/reference/pkg/src/wavefuse/bench.py:39-47): numpy PCG64 uniform
  [0, 255) float32, PAN drawn first, then each half-size band. Host-side;
  used for the reference-shaped bench config and parity tests.

* a counter-based hash (`hash_plane` on the host, `device_plane` on the GPU
  through wf_synth_plane_f32) addressable per (seed, plane, row, col), so any
  window of a 65536^2 scene or of a 64-scene batch can be regenerated on the
  host bit-exactly without materialising the whole thing. The device kernel
  (csrc/transforms.cu synth_kernel) and `hash_plane` compute identical float32
  values (tests/test_synth.py).
"""

from __future__ import annotations

import numpy as np

DEFAULT_SEED = 42  # bench.py:24

_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SCALE = np.float32(255.0 / 16777216.0)


def synth_scene(w: int, h: int, bands: int = 3, seed: int = DEFAULT_SEED):
    """bench.py:39-47: uniform-noise PAN plus half-resolution bands."""
    rng = np.random.default_rng(seed)
    pan = rng.uniform(0.0, 255.0, (h, w)).astype(np.float32)
    ms = [rng.uniform(0.0, 255.0, (h // 2, w // 2)).astype(np.float32) for _ in range(bands)]
    return pan, ms


def hash_plane(seed: int, plane: int, rows, cols) -> np.ndarray:
    """Values of plane `plane` at absolute (rows x cols) index vectors."""
    rows = np.asarray(rows, dtype=np.uint64)[:, None]
    cols = np.asarray(cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        s = np.uint64(seed) * _PHI
        key = (np.uint64(plane) << np.uint64(48)) ^ (rows << np.uint64(24)) ^ cols
        z = s + key
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return (z >> np.uint64(40)).astype(np.float32) * _SCALE


def plane_id(scene: int, band: int) -> int:
    """Plane numbering: PAN of scene s is 8*s, band k is 8*s + 1 + k."""
    return 8 * scene + (0 if band < 0 else 1 + band)


def device_plane(out, seed: int, plane: int, row0: int = 0, col0: int = 0) -> None:
    """Fill a contiguous CUDA float32 tensor `out` (rows x cols) with the
    hash plane window starting at (row0, col0), on the GPU."""
    from . import _device, _native

    rows, cols = out.shape
    _native.check(_native.load().wf_synth_plane_f32(
        out.data_ptr(), out.stride(0), rows, cols, seed, plane, row0, col0,
        _device.stream_ptr()))
