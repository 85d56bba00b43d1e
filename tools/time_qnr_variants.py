"""CUDA-event time of the one-pass QNR report (wf_quality_scene_f32) on a
fused Landsat-shaped scene for each scene kernel (WF_QNR_KERNEL = v3 default,
v2 role-split, v1 one-warp-per-block), with the report's values in hex so a
change of arithmetic is visible."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import _device, _native
from paper_1803_00737_b200.scene import DeviceScene

if os.environ.get("WF_LIB"):  # A/B: time another build of the library
    import pathlib
    _native.LIB_PATH = pathlib.Path(os.environ["WF_LIB"]).resolve()
    print(f"library: {_native.LIB_PATH.name}")

h = int(sys.argv[1]) if len(sys.argv) > 1 else 14000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16000
B = 6
scene = DeviceScene.synthetic(h, w, B)
scene.launcher(wf.WaveletKind.DAUB4)()
torch.cuda.synchronize()
lib = _native.load()
ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(B, h, w)) // 8 + 1,
                 dtype=torch.float64, device="cuda")
out = torch.zeros(64, dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
fp = _native.ptr_array([t.data_ptr() for t in scene.out])
mp = _native.ptr_array([t.data_ptr() for t in scene.ms])
nbytes = (4 * B + 4 + B) * h * w
for variant in (sys.argv[3:] or ["", "v2", "v1"]):
    os.environ["WF_QNR_KERNEL"] = variant
    _native.reload_tuning()

    def launch():
        _native.check(lib.wf_quality_scene_f32(fp, mp, scene.pan.data_ptr(), w, w // 2, w, B, h,
                                               w, ws.data_ptr(), out.data_ptr(), flag.data_ptr(),
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
    rep = wf.qnr(scene.out, scene.ms, scene.pan)
    print(f"{variant or 'v3'}: {ms:.3f} ms/report, {nbytes / ms / 1e6:.0f} GB/s; qnr={rep.qnr!r} "
          f"({rep.qnr.hex()}) ergas={rep.ergas!r} d_lambda={rep.d_lambda!r} d_s={rep.d_s!r} "
          f"flag={int(flag.item())}", flush=True)
