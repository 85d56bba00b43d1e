"""Time the 8 bpp kernels on the Landsat scene: Haar, and D4 per kernel variant
(WF_D4_U8), row-run length (WF_D4_PAIRS) and ring depth (WF_D4_STAGES)."""
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
# argv: configs "variant:pairs:stages" (0 = launcher default); D4 only when given
configs = sys.argv[1:] or ["haar", "v3:0:0", "v2:0:0", "v3:8:0", "v3:32:0"]
for cfg in configs:
    if cfg == "haar":
        kind, variant, p, st = 1, "v2", 0, 0
    else:
        variant, p, st = cfg.split(":")
        kind, p, st = 2, int(p), int(st)
    os.environ["WF_D4_U8"] = variant
    os.environ["WF_D4_PAIRS"] = str(p)
    os.environ["WF_D4_STAGES"] = str(st)
    _native.reload_tuning()
    if True:
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
        print(f"u8 {cfg}: {t:.3f} ms {nbytes / t / 1e6:.0f} GB/s "
              f"{H * W / t / 1e3:.0f} MPix/s", flush=True)
