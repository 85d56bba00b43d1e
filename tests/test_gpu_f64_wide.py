"""float64 callers (the reference's dtype for float64 numpy inputs,
fusion.py:46-47): rows whose starts are 32-byte aligned take 256-bit loads
and stores (LDG/STG.256), 16-byte aligned ones the 128-bit path. Both must
give the same bits, and match the float64 oracle."""
import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from oracle import cpu_dwt as O

pytestmark = pytest.mark.gpu


def _offset16(t):
    """The same values, contiguous, in a buffer that starts 16 bytes past a
    32-byte boundary (so with W * 8 % 32 == 0 every row start is 16- but not
    32-byte aligned)."""
    h, w = t.shape
    buf = torch.empty(h * w + 2, dtype=t.dtype, device=t.device)
    v = buf[2:].view(h, w)
    v.copy_(t)
    assert v.data_ptr() % 32 == 16
    return v


@pytest.mark.parametrize("kname", ["haar", "daub4"])
@pytest.mark.parametrize("shape,nb", [((64, 1024), 6), ((48, 520), 3), ((32, 4096), 1)])
def test_f64_wide_and_narrow_paths_agree(kname, shape, nb):
    rng = np.random.default_rng(5)
    h, w = shape
    pan = rng.uniform(0, 255, (h, w))
    ms = [rng.uniform(0, 255, (h // 2, w // 2)) for _ in range(nb)]
    kind = wf.WaveletKind.HAAR if kname == "haar" else wf.WaveletKind.DAUB4
    pd = torch.from_numpy(pan).cuda()
    md = [torch.from_numpy(m).cuda() for m in ms]
    wide = wf.fuse(pd, md, wf.DwtReplace(kind))
    narrow = wf.fuse(_offset16(pd), [_offset16(m) for m in md], wf.DwtReplace(kind))
    ref = O.fuse(pan, ms, kname)
    for a, b, r in zip(wide, narrow, ref):
        assert a.dtype == torch.float64
        assert torch.equal(a, b)
        assert np.max(np.abs(a.cpu().numpy() - r)) <= 1e-9
