"""Warm-up + profiled launches of an 8 bpp fusion kernel on the Landsat scene
(argv[1]: 1 = Haar, 2 = D4; default D4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import _native
from paper_1803_00737_b200.fusion import _quantize_dev
from paper_1803_00737_b200.scene import DeviceScene

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)
pan = _quantize_dev(sc.pan)
ms = [_quantize_dev(m) for m in sc.ms]
out = [torch.empty((H, W), dtype=torch.uint8, device="cuda") for _ in ms]
lib = _native.load()
mp = _native.ptr_array([m.data_ptr() for m in ms])
op = _native.ptr_array([o.data_ptr() for o in out])
KIND = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(2):
    _native.check(lib.wf_fuse_bands_u8(KIND, pan.data_ptr(), W, mp, W // 2, op, W, B, H, W, None))
torch.cuda.synchronize()
print("profile_u8 ok")
