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


class FuseScorePipeline:
    """Fusion and the QNR/ERGAS report of a sequence of scenes on two CUDA
    streams (the C5 batch): scene k's report (issue-bound,
    about half the HBM bandwidth) runs while scene k+1 fuses (HBM-bound, few
    issue slots), on two output sets used in turn. Each submit() queues one
    fusion launch and one report; the reports' scalars are read later, once,
    through the returned PendingReport (metrics.qnr_async), so the GPU never
    idles on a host sync. Same kernels and results as fuse() then qnr().

    Stream order: the fusion into output set k % 2 waits for the report that
    last read that set; the report waits for its fusion. wait() makes the
    caller's current stream wait for everything submitted."""

    def __init__(self, shape, bands: int, device=None):
        dev = _device.require_cuda() if device is None else device
        h, w = shape
        self.outs = [[torch.empty((h, w), dtype=torch.float32, device=dev) for _ in range(bands)]
                     for _ in range(2)]
        self.s_fuse = torch.cuda.Stream(device=dev)
        self.s_score = torch.cuda.Stream(device=dev)
        self.fused = [torch.cuda.Event(), torch.cuda.Event()]
        self.scored = [torch.cuda.Event(), torch.cuda.Event()]
        self.k = 0
        self.started = False

    def submit(self, scene: "DeviceScene", kind: WaveletKind):
        from .metrics import qnr_async

        if not self.started:  # nothing before this point on the caller's stream is skipped
            cur = torch.cuda.current_stream()
            self.s_fuse.wait_stream(cur)
            self.s_score.wait_stream(cur)
            self.started = True
        slot = self.k % 2
        outs = self.outs[slot]
        lib = _native.load()
        h, w = scene.shape
        self.s_fuse.wait_event(self.scored[slot])
        _native.check(lib.wf_fuse_bands_f32(
            KIND_CODE[kind], scene.pan.data_ptr(), w,
            _native.ptr_array([m.data_ptr() for m in scene.ms]), w // 2,
            _native.ptr_array([o.data_ptr() for o in outs]), w, len(scene.ms), h, w,
            self.s_fuse.cuda_stream))
        self.fused[slot].record(self.s_fuse)
        self.s_score.wait_event(self.fused[slot])
        with torch.cuda.stream(self.s_score):
            pending = qnr_async(outs, scene.ms, scene.pan)
        self.scored[slot].record(self.s_score)
        self.k += 1
        return pending

    def wait(self) -> None:
        cur = torch.cuda.current_stream()
        cur.wait_stream(self.s_fuse)
        cur.wait_stream(self.s_score)
        self.started = False
