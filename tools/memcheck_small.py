"""Small-shape exercise of every kernel, for compute-sanitizer (memcheck,
racecheck, synccheck): the fused kernels (Haar, D4 bulk-copy and register
paths, float64, strips, reference-exact), the transforms, the resample, the
8 bpp kernels (v3 byte-exact with every fix-up path, v2, v1), the QNR scene
kernels (v2 default, v3, v1, per-pair) and the one-pass fuse + report.

    compute-sanitizer --tool memcheck python tools/memcheck_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import _native, strips


def env(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    _native.reload_tuning()


rng = np.random.default_rng(1)
for (h, w, nb) in [(64, 1040, 6), (96, 200, 3), (8, 16, 2), (130, 264, 8), (6, 10, 1), (64, 64, 2)]:
    pan = torch.from_numpy(rng.uniform(0, 255, (h, w)).astype(np.float32)).cuda()
    ms = [torch.from_numpy(rng.uniform(1, 255, (h // 2, w // 2)).astype(np.float32)).cuda()
          for _ in range(nb)]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        for path in ("auto", "ldg"):
            env(WF_D4_PATH=path)
            out = wf.fuse(pan, ms, wf.DwtReplace(kind))
        env(WF_D4_PATH=None)
        wf.fuse(pan, ms, wf.DwtReplace(kind), exact=True)
        strips.fuse_scene_strips(kind, pan, ms)
        wf.fuse(pan.double(), [m.double() for m in ms], wf.DwtReplace(kind))
        if nb >= 2 and h >= 4:
            for qp in ("v2", "v3", "v1", "generic"):
                env(WF_QNR_PATH="generic" if qp == "generic" else None,
                    WF_QNR_KERNEL=None if qp == "generic" else qp)
                wf.qnr(out, ms, pan)
            env(WF_QNR_PATH=None, WF_QNR_KERNEL=None)
            if kind is wf.WaveletKind.HAAR:
                wf.fuse_and_qnr(pan, ms, wf.DwtReplace(kind), one_pass=True)
    if min(h, w) >= 4:
        c = wf.dwt2d_forward(pan, wf.WaveletKind.DAUB4)
        wf.dwt2d_inverse(c, wf.WaveletKind.DAUB4)
    wf.resample_bilinear(ms[0], w, h)
# 8 bpp kernels (W % 32 == 0): v3 (default, each fix-up path), v2 and v1 D4,
# Haar; device and host (strip) paths
for (h, w, nb) in [(64, 1056, 6), (34, 3104, 8), (4, 32, 2), (96, 2080, 3), (130, 1024, 1)]:
    pan8 = rng.integers(0, 256, (h, w), dtype=np.uint8)
    ms8 = [rng.integers(0, 256, (h // 2, w // 2), dtype=np.uint8) for _ in range(nb)]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        for v, fix in (("v3", None), ("v3", "all"), ("v3", "ref"), ("v2", None), ("v1", None)):
            env(WF_D4_U8=v, WF_U8_FIX=fix)
            wf.fuse_quantized(torch.from_numpy(pan8).cuda(),
                              [torch.from_numpy(m).cuda() for m in ms8], wf.DwtReplace(kind))
            wf.fuse_quantized(pan8, ms8, wf.DwtReplace(kind))
        env(WF_D4_U8=None, WF_U8_FIX=None)
host = wf.fuse(np.ones((130, 264), np.float32), [np.ones((65, 132), np.float32)] * 3,
               wf.DwtReplace(wf.WaveletKind.DAUB4))
torch.cuda.synchronize()
print("memcheck_small ok")
