"""Sweep Haar pairs-per-thread on the Landsat scene (f32, B bands)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1803_00737_b200 import WaveletKind
from paper_1803_00737_b200.scene import DeviceScene, scene_bytes

H, W = 14000, 16000
B = int(os.environ.get("SWEEP_BANDS", "6"))
scene = DeviceScene.synthetic(H, W, B)
nbytes = scene_bytes(H, W, B)
run = scene.launcher(WaveletKind.HAAR)
for ppt in [int(x) for x in sys.argv[1:]] or [4]:
    os.environ["WF_HAAR_PPT"] = str(ppt)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(30):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    print(f"haar B={B} ppt={ppt}: {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
