"""Diagnose the overlapped fuse + report on a small scene: WF_FQ_DEBUG=1
(banded fusion only) and 2 (report after the fusion), each in a fresh
process, compared with fuse() + the scene report."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1803_00737_b200 import WaveletKind, _device, _native  # noqa: E402
from paper_1803_00737_b200.scene import DeviceScene  # noqa: E402

h, w = int(sys.argv[1]), int(sys.argv[2])
code = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lib = _native.load()
scene = DeviceScene.synthetic(h, w, 6)
nb = 6
ws = torch.zeros(int(lib.wf_quality_scene_workspace_bytes(nb, h, w)) // 8 + 1,
                 dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
mp = _native.ptr_array([t.data_ptr() for t in scene.ms])
fp = _native.ptr_array([t.data_ptr() for t in scene.out])
scene.launcher(WaveletKind.HAAR if code == 1 else WaveletKind.DAUB4)()
ref = torch.zeros(64, dtype=torch.float64, device="cuda")
_native.check(lib.wf_quality_scene_f32(fp, mp, scene.pan.data_ptr(), w, w // 2, w, nb, h, w,
                                       ws.data_ptr(), ref.data_ptr(), flag.data_ptr(),
                                       _device.stream_ptr()))
torch.cuda.synchronize()
fo = [torch.zeros_like(scene.pan) for _ in scene.ms]
fop = _native.ptr_array([t.data_ptr() for t in fo])
out = torch.zeros(64, dtype=torch.float64, device="cuda")
_native.check(lib.wf_fuse_quality_f32(code, scene.pan.data_ptr(), w, mp, w // 2, fop, w, nb, h, w,
                                      ws.data_ptr(), out.data_ptr(), flag.data_ptr(),
                                      _device.stream_ptr()))
torch.cuda.synchronize()
for k, (a, b) in enumerate(zip(fo, scene.out)):
    d = (a - b).abs()
    bad = torch.nonzero(d > 0)
    print("band", k, "identical", bool(torch.equal(a, b)), "maxdiff", float(d.max()),
          "first bad", bad[:4].tolist())
print("report identical", bool(torch.equal(out, ref)), "maxdiff", float((out - ref).abs().max()))
print("undecidable flag", int(flag.item()))
