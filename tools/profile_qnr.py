"""Two launches of the scene-quality kernel sequence on the Landsat scene
(the command ncu wraps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

scene = DeviceScene.synthetic(14000, 16000, 6)
scene.launcher(wf.WaveletKind.HAAR)()
for _ in range(2):
    wf.qnr(scene.out, scene.ms, scene.pan)
torch.cuda.synchronize()
print("profile_qnr ok")
