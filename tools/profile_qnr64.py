"""Warm-up + profiled launches of the float64 one-pass QNR report on a
float64 Landsat-shaped D4 scene (the command ncu wraps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

sc = DeviceScene.synthetic(14000, 16000, 6)
pan = sc.pan.double()
ms = [m.double() for m in sc.ms]
del sc
torch.cuda.empty_cache()
fused = wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
for _ in range(2):
    wf.qnr(fused, ms, pan)
torch.cuda.synchronize()
print("profile_qnr64 ok")
