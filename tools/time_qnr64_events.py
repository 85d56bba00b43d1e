"""CUDA-event time of the float64 one-pass QNR report (wf_quality_scene_f64)
on a float64 Landsat-shaped scene fused with D4, and the report's hex values
(WF_LIB: time another build of the library)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_00737_b200 import _native  # noqa: E402

if os.environ.get("WF_LIB"):
    import pathlib
    _native.LIB_PATH = pathlib.Path(os.environ["WF_LIB"]).resolve()
import paper_1803_00737_b200 as wf  # noqa: E402
from paper_1803_00737_b200 import _device  # noqa: E402
from paper_1803_00737_b200.scene import DeviceScene  # noqa: E402

h, w, nb = 14000, 16000, 6
sc = DeviceScene.synthetic(h, w, nb)
pan = sc.pan.double()
ms = [m.double() for m in sc.ms]
del sc
torch.cuda.empty_cache()
fused = wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
lib = _native.load()
ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(nb, h, w)) // 8 + 1,
                 dtype=torch.float64, device="cuda")
out = torch.zeros(64, dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
fp = _native.ptr_array([t.data_ptr() for t in fused])
mp = _native.ptr_array([t.data_ptr() for t in ms])


def run():
    _native.check(lib.wf_quality_scene_f64(fp, mp, pan.data_ptr(), w, w // 2, w, nb, h, w,
                                           ws.data_ptr(), out.data_ptr(), flag.data_ptr(),
                                           _device.stream_ptr()))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
ms_per = e0.elapsed_time(e1) / 10
rep = wf.qnr(fused, ms, pan)
print(json.dumps({"ms_per_report": round(ms_per, 4), "qnr": rep.qnr.hex(), "ergas": rep.ergas.hex(),
                  "d_lambda": rep.d_lambda.hex()}))
