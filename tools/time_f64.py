"""Device-resident time of the float64 fused kernels (the reference's dtype for
float64 callers) on the Landsat scene: PAN 14000x16000 + 6 bands, f64 in/out,
(8 + 10*B) bytes per PAN px. Also the reference-exact mode (exact=True) per
band for comparison."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import _native
from paper_1803_00737_b200.scene import DeviceScene

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)
pan = sc.pan.double()
ms = [m.double() for m in sc.ms]
del sc
torch.cuda.empty_cache()
out = [torch.empty((H, W), dtype=torch.float64, device="cuda") for _ in ms]
lib = _native.load()
mp = _native.ptr_array([m.data_ptr() for m in ms])
op = _native.ptr_array([o.data_ptr() for o in out])
nbytes = (8 + 10 * B) * H * W


def timed(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


# argv: configs "haar:PPT" / "daub4:PAIRS:STAGES" / "daub4ldg" (0 = default)
configs = sys.argv[1:] or ["haar:0", "daub4:0:0", "daub4ldg"]
for cfg in configs:
    parts = cfg.split(":")
    name = parts[0]
    kind = 1 if name == "haar" else 2
    for k in ("WF_HAAR_PPT", "WF_D4_PAIRS", "WF_D4_STAGES", "WF_D4_PATH"):
        os.environ.pop(k, None)
    if name == "haar" and len(parts) > 1:
        os.environ["WF_HAAR_PPT"] = parts[1]
    if name == "daub4":
        if len(parts) > 1:
            os.environ["WF_D4_PAIRS"] = parts[1]
        if len(parts) > 2:
            os.environ["WF_D4_STAGES"] = parts[2]
    if name == "daub4ldg":
        os.environ["WF_D4_PATH"] = "ldg"
    t = timed(lambda: _native.check(lib.wf_fuse_bands_f64(kind, pan.data_ptr(), W, mp, W // 2,
                                                          op, W, B, H, W, None)))
    print(f"f64 {cfg}: {t:.3f} ms  {nbytes / t / 1e6:.0f} GB/s  "
          f"{H * W / t / 1e3:.0f} scene-MPix/s", flush=True)
