"""Time the numpy (pageable host memory) drop-in path on a Landsat-shaped
scene, single caller and 4 concurrent callers on quarter tiles."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1803_00737_b200 as wf
from paper_1803_00737_b200 import synth

H, W, B = 14000, 16000, 6
pan = synth.hash_plane(42, 0, np.arange(H), np.arange(W))
ms = [synth.hash_plane(42, 1 + b, np.arange(H // 2), np.arange(W // 2)) for b in range(B)]
for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
    m = wf.DwtReplace(kind)
    wf.fuse(pan[:512], [b[:256] for b in ms], m)
    for rep in range(4):
        t0 = time.perf_counter()
        wf.fuse(pan, ms, m)
        dt = time.perf_counter() - t0
        print(f"{kind.value} numpy fuse 1 caller: {dt * 1e3:.1f} ms = {H * W / dt / 1e6:.0f} "
              f"scene-MPix/s", flush=True)
    quarters = [(pan[r:r + H // 4], [b[r // 2:(r + H // 4) // 2] for b in ms])
                for r in range(0, H, H // 4)]
    with ThreadPoolExecutor(4) as ex:
        list(ex.map(lambda q: wf.fuse(q[0], q[1], m), quarters))
        for rep in range(3):
            t0 = time.perf_counter()
            list(ex.map(lambda q: wf.fuse(q[0], q[1], m), quarters))
            dt = time.perf_counter() - t0
            print(f"{kind.value} numpy fuse 4 callers x quarter scene: {dt * 1e3:.1f} ms = "
                  f"{H * W / dt / 1e6:.0f} scene-MPix/s", flush=True)
