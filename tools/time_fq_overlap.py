"""Fusion + report in one call (wf_fuse_quality_f32): the default schedule
(Haar one pass; D4 fusion then report) and, with WF_FQ_OVERLAP=1, the
SM-partitioned overlap (fusion in row bands on an internal stream, the report
kernel on fewer persistent CTAs scoring each band as it lands) against fuse() + qnr() on a Landsat-shaped scene, Haar and D4,
over a sweep of report CTAs (WF_FQ_CTAS) and band rows (WF_FQ_BAND_ROWS).
Each line: CUDA-event ms per fused + scored scene, and whether the fused bands
and the report vector are bit-identical to the two separate calls.

    python tools/time_fq_overlap.py [H W] [--quick]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1803_00737_b200 import WaveletKind, _device, _native  # noqa: E402
from paper_1803_00737_b200.scene import DeviceScene  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
h = int(args[0]) if args else 14000
w = int(args[1]) if len(args) > 1 else 16000
quick = "--quick" in sys.argv
lib = _native.load()
scene = DeviceScene.synthetic(h, w, 6)
nb = len(scene.ms)
ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(nb, h, w)) // 8 + 1,
                 dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
mp = _native.ptr_array([t.data_ptr() for t in scene.ms])
fp = _native.ptr_array([t.data_ptr() for t in scene.out])
fo = [torch.empty_like(scene.pan) for _ in scene.ms]
fop = _native.ptr_array([t.data_ptr() for t in fo])


def timed(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def set_env(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = str(v)
    lib.wf_tuning_reload()


for kind, name in ((WaveletKind.DAUB4, "daub4"), (WaveletKind.HAAR, "haar")):
    code = 1 if kind == WaveletKind.HAAR else 2
    set_env(WF_FQ_CTAS=None, WF_FQ_BAND_ROWS=None, WF_FQ_OVERLAP=None)
    fuse = scene.launcher(kind)
    ref_out = torch.zeros(64, dtype=torch.float64, device="cuda")

    def score(out=ref_out):
        _native.check(lib.wf_quality_scene_f32(fp, mp, scene.pan.data_ptr(), w, w // 2, w, nb, h,
                                               w, ws.data_ptr(), out.data_ptr(),
                                               flag.data_ptr(), _device.stream_ptr()))

    t_fuse = timed(fuse)
    t_score = timed(score)
    t_both = timed(lambda: (fuse(), score()))
    print(json.dumps({"kind": name, "fuse_ms": round(t_fuse, 4), "qnr_ms": round(t_score, 4),
                      "fuse_then_qnr_ms": round(t_both, 4)}), flush=True)
    ref_bands = [t.clone() for t in scene.out]
    ref_rep = ref_out.clone()
    out = torch.zeros(64, dtype=torch.float64, device="cuda")

    def fused():
        _native.check(lib.wf_fuse_quality_f32(code, scene.pan.data_ptr(), w, mp, w // 2, fop, w,
                                              nb, h, w, ws.data_ptr(), out.data_ptr(),
                                              flag.data_ptr(), _device.stream_ptr()))

    if True:  # the default schedule: Haar one pass, D4 fusion then report
        t = timed(fused)
        same = all(torch.equal(a, b) for a, b in zip(fo, ref_bands))
        print(json.dumps({"kind": name, "mode": "default", "ms": round(t, 4),
                          "bands_identical": same,
                          "report_identical": bool(torch.equal(out, ref_rep))}), flush=True)
    def opt(name, default):
        for a in sys.argv:
            if a.startswith(f"--{name}="):
                return [int(x) for x in a.split("=", 1)[1].split(",")]
        return default

    ctas = [120] if quick else opt("ctas", [100, 110, 116, 120, 124, 128, 134])
    bands = [512] if quick else opt("bands", [256, 512, 1024])
    stages = opt("stages", [0])
    for c, br, st in [(c, br, st) for c in ctas for br in bands for st in stages]:
            set_env(WF_FQ_CTAS=c, WF_FQ_BAND_ROWS=br, WF_D4_STAGES=st or None, WF_FQ_OVERLAP=1)
            for o in fo:
                o.zero_()
            out.zero_()
            t = timed(fused)
            same = all(torch.equal(a, b) for a, b in zip(fo, ref_bands))
            print(json.dumps({"kind": name, "mode": "overlap", "ctas": c, "band_rows": br,
                              "d4_stages": st,
                              "ms": round(t, 4), "bands_identical": same,
                              "report_identical": bool(torch.equal(out, ref_rep))}), flush=True)
