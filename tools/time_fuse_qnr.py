"""One-pass Haar fusion + QNR report (wf_fuse_quality_f32, SURVEY.md 8(f)
row f1) against fuse() + qnr() on a Landsat-shaped scene: bench.py's
measure_quality, printed as JSON (CUDA events; set WF_LIB to A/B another
build of the library)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1803_00737_b200 import _native  # noqa: E402

if os.environ.get("WF_LIB"):
    import pathlib
    _native.LIB_PATH = pathlib.Path(os.environ["WF_LIB"]).resolve()

import bench  # noqa: E402
from paper_1803_00737_b200.scene import DeviceScene  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 14000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16000
scene = DeviceScene.synthetic(h, w, 6)
q = bench.measure_quality(scene, 10, 3, 6546.9)
print(json.dumps({"ms_per_report": q["ms_per_report"], **q["fused_haar_fuse_and_report"],
                  "report": q["report"]}))
