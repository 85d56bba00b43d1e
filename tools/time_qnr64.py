"""CUDA-event time of the float64 one-pass QNR report (wf_quality_scene_f64)
on a float64 Landsat-shaped scene fused with D4, next to the per-pair float64
kernels (WF_QNR_PATH=generic), with both reports."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import _native
from paper_1803_00737_b200.scene import DeviceScene

h = int(sys.argv[1]) if len(sys.argv) > 1 else 14000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16000
sc = DeviceScene.synthetic(h, w, 6)
pan = sc.pan.double()
ms = [m.double() for m in sc.ms]
del sc
torch.cuda.empty_cache()
fused = wf.fuse(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
for path in ("scene", "generic"):
    os.environ.pop("WF_QNR_PATH", None)
    if path == "generic":
        os.environ["WF_QNR_PATH"] = "generic"
    wf.qnr(fused, ms, pan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n0 = _native.launch_count()
    reps = 5 if path == "scene" else 2
    for _ in range(reps):
        r = wf.qnr(fused, ms, pan)
    torch.cuda.synchronize()
    ms_ = 1e3 * (time.perf_counter() - t0) / reps
    print(f"{path}: {ms_:.2f} ms/report wall ({(_native.launch_count() - n0) // reps} launches) "
          f"ergas={r.ergas!r} qnr={r.qnr!r} d_l={r.d_lambda!r} d_s={r.d_s!r}", flush=True)
