"""Two calls of the one-pass Haar fusion + quality report on the Landsat
scene (the command ncu wraps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

scene = DeviceScene.synthetic(14000, 16000, 6)
for _ in range(2):
    wf.fuse_and_qnr(scene.pan, scene.ms, wf.DwtReplace(wf.WaveletKind.HAAR))
torch.cuda.synchronize()
print("profile_fused_qnr ok")
