"""Time the GPU QNR report on a fused scene (device tensors)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

h = int(sys.argv[1]) if len(sys.argv) > 1 else 14000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16000
scene = DeviceScene.synthetic(h, w, 6)
scene.launcher(wf.WaveletKind.HAAR)()
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    r = wf.qnr(scene.out, scene.ms, scene.pan)
    torch.cuda.synchronize()
    print(f"qnr {h}x{w}x6: {time.perf_counter() - t0:.3f} s  ergas={r.ergas:.6f} "
          f"qnr={r.qnr:.6f} d_l={r.d_lambda:.6f} d_s={r.d_s:.6f}", flush=True)
