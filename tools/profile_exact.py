"""Two launches of the one-pass reference-exact D4 (argv[1] = 2) or Haar (1)
fusion on the Landsat scene (the command ncu wraps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene

kind = wf.WaveletKind.DAUB4 if (sys.argv[1:] or ["2"])[0] == "2" else wf.WaveletKind.HAAR
sc = DeviceScene.synthetic(14000, 16000, 6)
for _ in range(2):
    wf.fuse(sc.pan, sc.ms, wf.DwtReplace(kind), exact=True)
torch.cuda.synchronize()
print("profile_exact ok")
