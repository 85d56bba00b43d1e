"""Time the GPU QNR report on a fused Landsat-shaped scene (device tensors):
wall time of wf.qnr and CUDA-event time of the scene-kernel launch sequence."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import _device, _native
from paper_1803_00737_b200.scene import DeviceScene

h = int(sys.argv[1]) if len(sys.argv) > 1 else 14000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16000
B = 6
scene = DeviceScene.synthetic(h, w, B)
scene.launcher(wf.WaveletKind.HAAR)()
torch.cuda.synchronize()
for path in ("scene", "generic"):
    if path == "generic":
        os.environ["WF_QNR_PATH"] = "generic"
    for rep in range(3):
        t0 = time.perf_counter()
        r = wf.qnr(scene.out, scene.ms, scene.pan)
        torch.cuda.synchronize()
        print(f"{path} qnr {h}x{w}x{B}: {1e3 * (time.perf_counter() - t0):.2f} ms wall  "
              f"ergas={r.ergas:.6f} qnr={r.qnr:.6f} d_l={r.d_lambda:.6f} d_s={r.d_s:.6f}",
              flush=True)
os.environ.pop("WF_QNR_PATH")
lib = _native.load()
ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(B, h, w)) // 8 + 1,
                 dtype=torch.float64, device="cuda")
out = torch.zeros(64, dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
fp = _native.ptr_array([t.data_ptr() for t in scene.out])
mp = _native.ptr_array([t.data_ptr() for t in scene.ms])


def launch():
    _native.check(lib.wf_quality_scene_f32(fp, mp, scene.pan.data_ptr(), w, w // 2, w, B, h, w,
                                           ws.data_ptr(), out.data_ptr(), flag.data_ptr(),
                                           _device.stream_ptr()))


for _ in range(3):
    launch()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    launch()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nbytes = (4 * B + 4 + B) * h * w
print(f"scene kernel sequence: {ms:.3f} ms/report, {nbytes / ms / 1e6:.0f} GB/s of "
      f"{nbytes / 1e9:.2f} GB algorithmic", flush=True)
