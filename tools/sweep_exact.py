"""Coefficient rows per CTA (WF_EXACT_ROWS) of the one-pass reference-exact D4
kernel on the Landsat scene (f32 planes): CUDA-event time per scene. A run of
R coefficient rows re-reads 4 PAN rows and 1 MS row of halo, (4 / 2R) and
(1 / R) of the plane, and redoes their row passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import _native

if os.environ.get("WF_LIB"):  # A/B: time another build of the library
    import pathlib
    _native.LIB_PATH = pathlib.Path(os.environ["WF_LIB"]).resolve()
from paper_1803_00737_b200.scene import DeviceScene

H, W, B = 14000, 16000, 6
sc = DeviceScene.synthetic(H, W, B)
lib = _native.load()
mp = _native.ptr_array([m.data_ptr() for m in sc.ms])
op = _native.ptr_array([o.data_ptr() for o in sc.out])
ws = torch.empty(1, dtype=torch.float64, device="cuda")
ref = None
for rows in (sys.argv[1:] or ["16", "32", "64", "128"]):
    os.environ["WF_EXACT_ROWS"] = rows
    _native.reload_tuning()

    def run():
        _native.check(lib.wf_fuse_bands_exact_f32(2, sc.pan.data_ptr(), W, mp, W // 2, op, W, B,
                                                  H, W, ws.data_ptr(), None))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    same = True
    if ref is None:
        ref = [o.clone() for o in sc.out]
    else:
        same = all(torch.equal(a, b) for a, b in zip(ref, sc.out))
    print(f"exact D4 rows={rows}: {t:.3f} ms, {(4 + 5 * B) * H * W / t / 1e6:.0f} GB/s, "
          f"identical={same}", flush=True)
