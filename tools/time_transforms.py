"""Device-resident times of the standalone transform API on a Landsat-sized
plane (14000 x 16000): dwt2d_forward / dwt2d_inverse (float64 arithmetic in
the reference's operation order, wavelet.py:149-164), resample_bilinear (2x),
and the reference-exact fusion (exact=True) of a 6-band scene."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for dt in (torch.float32, torch.float64):
    pan = sc.pan.to(dt)
    esz = pan.element_size()
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        c = wf.dwt2d_forward(pan, kind)
        t = timed(lambda: wf.dwt2d_forward(pan, kind))
        print(f"dwt2d_forward {dt} {kind.value}: {t:.3f} ms  {2 * esz * H * W / t / 1e6:.0f} GB/s",
              flush=True)
        t = timed(lambda: wf.dwt2d_inverse(c, kind))
        print(f"dwt2d_inverse {dt} {kind.value}: {t:.3f} ms  {2 * esz * H * W / t / 1e6:.0f} GB/s",
              flush=True)
        del c
    m = sc.ms[0].to(dt)
    t = timed(lambda: wf.resample_bilinear(m, W, H))
    print(f"resample_bilinear {dt} 2x: {t:.3f} ms  {esz * 1.25 * H * W / t / 1e6:.0f} GB/s",
          flush=True)
    ms = [x.to(dt) for x in sc.ms]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        t = timed(lambda: wf.fuse(pan, ms, wf.DwtReplace(kind), exact=True), n=2)
        print(f"fuse exact=True {dt} {kind.value} (6 bands): {t:.3f} ms", flush=True)
    del pan, ms, m
    torch.cuda.empty_cache()
