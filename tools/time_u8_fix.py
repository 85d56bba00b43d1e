"""Split the byte-exact 8 bpp D4 kernel's time: full (detect + queue + the
in-ring float64 fix-up), detection without the fix-up (WF_U8_FIX=skipfix), no
detection (nodetect), and the round-1 v2 kernel; plus how many bytes the
fix-up changes (counted by diffing against the no-fix-up bytes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import _native

if len(sys.argv) > 1:  # A/B: time another build of the library
    import pathlib
    _native.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
    print(f"library: {sys.argv[1]}")
from paper_1803_00737_b200.fusion import _quantize_dev
from paper_1803_00737_b200.scene import DeviceScene

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)
pan = _quantize_dev(sc.pan)
ms = [_quantize_dev(m) for m in sc.ms]
del sc
lib = _native.load()
mp = _native.ptr_array([m.data_ptr() for m in ms])
res = {}
modes = (("v3", ""), ("v3", "skipfix"), ("v3", "nodetect"), ("v2", ""))
if os.environ.get("WF_TIME_MODES"):  # e.g. "v3:skipfix,v2:"
    modes = tuple(tuple(m.split(":")) for m in os.environ["WF_TIME_MODES"].split(","))
for variant, fix in modes:
    os.environ["WF_D4_U8"] = variant
    os.environ["WF_U8_FIX"] = fix
    _native.reload_tuning()
    out = [torch.empty((H, W), dtype=torch.uint8, device="cuda") for _ in ms]
    op = _native.ptr_array([o.data_ptr() for o in out])
    run = lambda: _native.check(lib.wf_fuse_bands_u8(2, pan.data_ptr(), W, mp, W // 2, op,  # noqa
                                                     W, B, H, W, None))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    print(f"{variant} {fix or 'full'}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    res[(variant, fix)] = out
if ("v3", "") not in res or ("v3", "skipfix") not in res or ("v2", "") not in res:
    sys.exit(0)
full, skip = res[("v3", "")], res[("v3", "skipfix")]
changed = sum(int((a != b).sum()) for a, b in zip(full, skip))
v2diff = sum(int((a != b).sum()) for a, b in zip(full, res[("v2", "")]))
print(f"bytes changed by the fix-up: {changed} of {B * H * W}; v3 vs v2 bytes differ: {v2diff}")
