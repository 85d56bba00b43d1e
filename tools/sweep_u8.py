"""Time the 8 bpp kernels on the Landsat scene for several D4 row-run lengths."""
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
nbytes = H * W + B * (H * W // 4 + H * W)
for kind, pairs in ((1, [0]), (2, [4, 8, 16, 32, 64])):
    for p in pairs:
        os.environ["WF_D4_PAIRS"] = str(p)
        run = lambda: _native.check(lib.wf_fuse_bands_u8(kind, pan.data_ptr(), W, mp, W // 2, op,
                                                         W, B, H, W, None))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20
        print(f"u8 kind={kind} pairs={p}: {t:.3f} ms {nbytes / t / 1e6:.0f} GB/s "
              f"{H * W / t / 1e3:.0f} MPix/s", flush=True)
