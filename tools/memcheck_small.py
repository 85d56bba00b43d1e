"""Small-shape exercise of every kernel, for compute-sanitizer memcheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import strips

rng = np.random.default_rng(1)
for (h, w, nb) in [(64, 1040, 6), (96, 200, 3), (8, 16, 2), (130, 264, 8), (6, 10, 1), (64, 64, 2)]:
    pan = torch.from_numpy(rng.uniform(0, 255, (h, w)).astype(np.float32)).cuda()
    ms = [torch.from_numpy(rng.uniform(1, 255, (h // 2, w // 2)).astype(np.float32)).cuda()
          for _ in range(nb)]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        for path in ("auto", "ldg"):
            os.environ["WF_D4_PATH"] = path
            out = wf.fuse(pan, ms, wf.DwtReplace(kind))
        os.environ.pop("WF_D4_PATH")
        strips.fuse_scene_strips(kind, pan, ms)
        wf.fuse(pan.double(), [m.double() for m in ms], wf.DwtReplace(kind))
        if nb >= 2 and h >= 4:
            for qp in ("scene", "generic"):
                if qp == "generic":
                    os.environ["WF_QNR_PATH"] = "generic"
                wf.qnr(out, ms, pan)
                os.environ.pop("WF_QNR_PATH", None)
    if min(h, w) >= 4:
        c = wf.dwt2d_forward(pan, wf.WaveletKind.DAUB4)
        wf.dwt2d_inverse(c, wf.WaveletKind.DAUB4)
    wf.resample_bilinear(ms[0], w, h)
# 8 bpp kernels (W % 32 == 0): v2 (default) and v1 D4, Haar, device and host paths
for (h, w, nb) in [(64, 1056, 6), (34, 3104, 8), (4, 32, 2), (96, 2080, 3), (130, 1024, 1)]:
    pan8 = rng.integers(0, 256, (h, w), dtype=np.uint8)
    ms8 = [rng.integers(0, 256, (h // 2, w // 2), dtype=np.uint8) for _ in range(nb)]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        for v in ("v2", "v1"):
            os.environ["WF_D4_U8"] = v
            wf.fuse_quantized(torch.from_numpy(pan8).cuda(),
                              [torch.from_numpy(m).cuda() for m in ms8], wf.DwtReplace(kind))
            wf.fuse_quantized(pan8, ms8, wf.DwtReplace(kind))
        os.environ.pop("WF_D4_U8")
host = wf.fuse(np.ones((130, 264), np.float32), [np.ones((65, 132), np.float32)] * 3,
               wf.DwtReplace(wf.WaveletKind.DAUB4))
torch.cuda.synchronize()
print("memcheck_small ok")
