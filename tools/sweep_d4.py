"""Sweep D4 launch geometry on the Landsat scene (device-resident, CUDA
events). Usage on the GPU box:
  python tools/sweep_d4.py [--haar] [--ldg] [pairs ...] [--stages s1,s2]"""
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
kind = WaveletKind.HAAR if "--haar" in sys.argv else WaveletKind.DAUB4
if "--ldg" in sys.argv:
    os.environ["WF_D4_PATH"] = "ldg"
stages = [0]
args = sys.argv[1:]
if "--stages" in args:
    stages = [int(x) for x in args[args.index("--stages") + 1].split(",")]
    del args[args.index("--stages"): args.index("--stages") + 2]
pairs = [int(a) for a in args if not a.startswith("--")] or [0]
run = scene.launcher(kind)
for st in stages:
    os.environ["WF_D4_STAGES"] = str(st)
    for p in pairs:
        os.environ["WF_D4_PAIRS"] = str(p)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 20
        e0.record()
        for _ in range(n):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{kind.value} B={B} {os.environ.get('WF_D4_PATH', 'auto')} stages={st} "
              f"pairs={p:5d}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
