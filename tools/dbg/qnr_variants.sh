#!/bin/bash
# A/B of the QNR scene kernel build variants in tools/dbg/lib_*.so against the
# in-tree library: timing (tools/time_qnr.py, scene path) and the report's
# float64 values (must be bit-identical), plus the GPU metric tests.
cd "$(dirname "$0")/../.."
LIB=paper_1803_00737_b200/libwavefuse_b200.so
cp $LIB /tmp/lib_base.so
for v in base tools/dbg/lib_*.so; do
  if [ $v = base ]; then cp /tmp/lib_base.so $LIB; name=base; else cp $v $LIB; name=$(basename $v .so); fi
  touch $LIB
  echo "=== $name"
  python - <<'PY'
import torch, paper_1803_00737_b200 as wf
from paper_1803_00737_b200.scene import DeviceScene
for (h, w) in ((14000, 16000), (1000, 1216)):
    s = DeviceScene.synthetic(h, w, 6)
    s.launcher(wf.WaveletKind.HAAR)()
    r = wf.qnr(s.out, s.ms, s.pan)
    print(h, w, [x.hex() for x in (r.ergas, r.qnr, r.d_lambda, r.d_s)])
PY
  WF_QNR_PATH= timeout 300 python tools/time_qnr.py 2>&1 | grep "scene kernel"
  timeout 600 python -m pytest tests/test_gpu_metrics.py -m gpu -x -q 2>&1 | tail -1
done
cp /tmp/lib_base.so $LIB
