"""Device-resident scenes and the throughput accounting of the hot path.

A *scene* is one PAN plane (H x W) plus B half-resolution MS bands, the unit
the reference's bench times (bench.py:50-61,100: MPix/s = PAN pixels / wall
time, all bands inside the timed region).

Algorithmic HBM bytes of one fused pass over a scene (the roofline
numerator, extended to the PAN-once multi-band
kernel of row f1): PAN read once (itemsize per px), each band's MS read
(itemsize / 4 per px) and fused write (itemsize per px):

    bytes(scene) = (1 + B * (1/4 + 1)) * itemsize * H * W
                 = (4 + 5B) * H * W  for float32 I/O  (34 B/px at B = 6)
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device, _native, synth
from .wavelet import KIND_CODE, WaveletKind


def scene_bytes(h: int, w: int, bands: int, itemsize: int = 4) -> int:
    return int(itemsize * h * w + bands * (itemsize * (h // 2) * (w // 2) + itemsize * h * w))


@dataclass
class DeviceScene:
    pan: torch.Tensor
    ms: list[torch.Tensor]
    out: list[torch.Tensor]

    @property
    def shape(self):
        return tuple(self.pan.shape)

    @classmethod
    def synthetic(cls, h: int, w: int, bands: int, seed: int = synth.DEFAULT_SEED,
                  scene: int = 0, outputs: bool = True) -> "DeviceScene":
        """Counter-hash planes generated on the device (no host round trip);
        outputs=False: no fused-band buffers (a pipeline brings its own)."""
        dev = _device.require_cuda()
        pan = torch.empty((h, w), dtype=torch.float32, device=dev)
        synth.device_plane(pan, seed, synth.plane_id(scene, -1))
        ms = []
        for b in range(bands):
            t = torch.empty((h // 2, w // 2), dtype=torch.float32, device=dev)
            synth.device_plane(t, seed, synth.plane_id(scene, b))
            ms.append(t)
        out = [torch.empty_like(pan) for _ in range(bands)] if outputs else []
        return cls(pan, ms, out)

    def launcher(self, kind: WaveletKind):
        """Return a zero-argument callable issuing ONE fused launch over the
        whole scene on the current stream (argument marshalling hoisted)."""
        lib = _native.load()
        h, w = self.shape
        ms_ptrs = _native.ptr_array([m.data_ptr() for m in self.ms])
        out_ptrs = _native.ptr_array([o.data_ptr() for o in self.out])
        fn = lib.wf_fuse_bands_f32
        code = KIND_CODE[kind]
        pan = self.pan.data_ptr()
        nb = len(self.ms)

        def run(stream: int | None = None):
            s = _device.stream_ptr() if stream is None else stream
            _native.check(fn(code, pan, w, ms_ptrs, w // 2, out_ptrs, w, nb, h, w, s))

        return run

