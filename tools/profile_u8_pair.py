"""One launch each of the byte-exact 8 bpp D4 pair (v3 + fix-up) and of the
round-1 v2 kernel on the Landsat scene, after one warm-up of each (the
command ncu wraps: -k regex:u8x8 -s 2 -c 2 captures v3 then v2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import _native
from paper_1803_00737_b200.fusion import _quantize_dev
from paper_1803_00737_b200.scene import DeviceScene

if os.environ.get("WF_LIB"):  # A/B: profile another build of the library
    import pathlib
    _native.LIB_PATH = pathlib.Path(os.environ["WF_LIB"]).resolve()

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)
pan = _quantize_dev(sc.pan)
ms = [_quantize_dev(m) for m in sc.ms]
del sc
out = [torch.empty((H, W), dtype=torch.uint8, device="cuda") for _ in ms]
lib = _native.load()
mp = _native.ptr_array([m.data_ptr() for m in ms])
op = _native.ptr_array([o.data_ptr() for o in out])
for rep in range(2):
    for v in ("v3", "v2"):
        os.environ["WF_D4_U8"] = v
        _native.reload_tuning()
        _native.check(lib.wf_fuse_bands_u8(2, pan.data_ptr(), W, mp, W // 2, op, W, B, H, W, None))
torch.cuda.synchronize()
print("profile_u8_pair ok")
