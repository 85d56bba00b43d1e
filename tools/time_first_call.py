"""First-call latencies of the drop-in (what a one-shot CLI-style caller
pays): CUDA context, library load, first fuse, first qnr, on the Landsat
scene from numpy."""
import os
import sys
import time

t_start = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1803_00737_b200 as wf  # noqa: E402
from paper_1803_00737_b200 import _native, synth  # noqa: E402


def lap(label, t0):
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    return time.perf_counter()


t = time.perf_counter()
print(f"imports: {1e3 * (t - t_start):.1f} ms", flush=True)
torch.cuda.init()
torch.empty(1, device="cuda")
t = lap("CUDA context", t)
_native.load()
t = lap("library load", t)
H, W, B = 14000, 16000, 6
pan = synth.hash_plane(42, 0, np.arange(H), np.arange(W))
ms = [synth.hash_plane(42, 1 + b, np.arange(H // 2), np.arange(W // 2)) for b in range(B)]
t = time.perf_counter()
for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
    for rep in range(2):
        fused = wf.fuse(pan, ms, wf.DwtReplace(kind))
        t = lap(f"fuse numpy {kind.value} call {rep + 1}", t)
for rep in range(2):
    wf.qnr(fused, ms, pan)
    t = lap(f"qnr numpy call {rep + 1}", t)
pd = torch.from_numpy(pan).cuda()
md = [torch.from_numpy(m).cuda() for m in ms]
fd = [torch.from_numpy(f).cuda() for f in fused]
t = lap("H2D of the scene (torch)", t)
for rep in range(2):
    wf.qnr(fd, md, pd)
    t = lap(f"qnr device call {rep + 1}", t)
# the rest of the numpy-facing API on the same scene
grid = wf.plan_grid(W, H, 4, 2)
for rep in range(2):
    wf.fuse_tiled(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4), grid)
    t = lap(f"fuse_tiled numpy 4x2 D4 call {rep + 1}", t)
for rep in range(2):
    c = wf.dwt2d_forward(pan, wf.WaveletKind.DAUB4)
    t = lap(f"dwt2d_forward numpy call {rep + 1}", t)
for rep in range(2):
    wf.dwt2d_inverse(c, wf.WaveletKind.DAUB4)
    t = lap(f"dwt2d_inverse numpy call {rep + 1}", t)
for rep in range(2):
    wf.resample_bilinear(ms[0], W, H)
    t = lap(f"resample_bilinear numpy 2x call {rep + 1}", t)
for rep in range(2):
    wf.fuse_and_qnr(pan, ms, wf.DwtReplace(wf.WaveletKind.DAUB4))
    t = lap(f"fuse_and_qnr numpy D4 call {rep + 1}", t)
