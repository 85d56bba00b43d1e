"""One warm-up + one profiled launch of each fused kernel on the Landsat
scene (PAN 14000x16000 + 6 bands, f32): the command ncu wraps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import WaveletKind
from paper_1803_00737_b200.scene import DeviceScene

scene = DeviceScene.synthetic(14000, 16000, 6)
for kind in (WaveletKind.HAAR, WaveletKind.DAUB4):
    run = scene.launcher(kind)
    run()
    run()
torch.cuda.synchronize()
print("profile_once ok")
