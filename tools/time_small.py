"""Wall-clock latency of one drop-in call on small numpy inputs (the
reference's tile sizes; configs[0] is 1024x1024 + 3 bands): fuse() through
the host pipeline, fast and exact, and qnr() on the result."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1803_00737_b200 as wf

rng = np.random.default_rng(42)
for (h, w, nb) in [(256, 256, 3), (1024, 1024, 3), (2048, 2048, 6)]:
    pan = rng.uniform(0, 255, (h, w)).astype(np.float32)
    ms = [rng.uniform(0, 255, (h // 2, w // 2)).astype(np.float32) for _ in range(nb)]
    for kind in (wf.WaveletKind.HAAR, wf.WaveletKind.DAUB4):
        for exact in (False, True):
            m = wf.DwtReplace(kind)
            wf.fuse(pan, ms, m, exact=exact)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                out = wf.fuse(pan, ms, m, exact=exact)
                ts.append(time.perf_counter() - t0)
            t = sorted(ts)[len(ts) // 2]
            print(f"fuse {h}x{w}x{nb} {kind.value} exact={exact}: {t * 1e3:.2f} ms "
                  f"({h * w / t / 1e6:.0f} scene-MPix/s)", flush=True)
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            wf.qnr(out, ms, pan)
            ts.append(time.perf_counter() - t0)
        print(f"qnr {h}x{w}x{nb}: {sorted(ts)[5] * 1e3:.2f} ms", flush=True)
