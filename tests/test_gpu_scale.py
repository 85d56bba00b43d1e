"""Parity at the sizes the bench reports.

* C4: one 65536 x 65536 D4 scene (17.2 GB PAN, elements beyond 2^31) on one
  GPU, fused whole and as 8 row strips through wf_fuse_strip_f32 whose halo
  pointers are the neighbouring strips' rows (what PeerHalos hands the kernel
  on 8 GPUs; rank 0 <-> rank 7 wrap): the strips equal the whole-scene launch
  bit for bit, and F4 windows at every seam, rows 0 and H-1, columns 0 and
  W-1 and past element 2^31 match the windowed oracle (1e-3 fast; the
  reference-exact strips bit for bit).
* C2/C3: the 6-band QNR report of a full Landsat scene through the one-pass
  scene kernel (float32 partials) against the per-pair float64 kernels
  (WF_QNR_PATH=generic, pinned to the reference's reports at 1e-9), and a
  2048 x 2048 crop of it against the oracle's qnr (the reference's
  metrics.py restated) -- all within 1e-6 (the north star asks 4 decimals).

The scene planes are the device counter-hash generator; the oracle rebuilds
any window of them on the host (synth.hash_plane), so nothing large crosses
PCIe.
"""

import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from oracle import cpu_dwt as O
from oracle import cpu_quality as Q
from paper_1803_00737_b200 import _native, synth

pytestmark = pytest.mark.gpu

SEED = 42


def _strips(fn, pan, ms, out, cuts):
    """wf_fuse_strip_* per strip [r0, r1) of the device scene, the halo rows
    pointing into the neighbouring strips (periodic: strip 0's top is the
    scene's last two rows)."""
    H, W = pan.shape
    es = pan.element_size()
    s = torch.cuda.current_stream().cuda_stream
    row = lambda t, r: t.data_ptr() + (r % t.shape[0]) * t.stride(0) * es  # noqa: E731
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        # the halo "buffers": rows r0-2, r0-1 and r1, r1+1 are consecutive in
        # the scene except across the wrap, where the caller's planes are
        # contiguous copies (only strip 0 / the last strip wrap)
        if r0 == 0:
            top = pan[[H - 2, H - 1]].contiguous()
            top_p, hp = top.data_ptr(), W
        else:
            top, top_p, hp = None, row(pan, r0 - 2), W
        if r1 == H:
            bot = pan[[0, 1]].contiguous()
            bot_p = bot.data_ptr()
        else:
            bot, bot_p = None, row(pan, r1)
        mtop = [row(m, r0 // 2 - 1) for m in ms]
        _native.check(fn(2, row(pan, r0), W, top_p, bot_p, hp,
                         _native.ptr_array([row(m, r0 // 2) for m in ms]),
                         _native.ptr_array(mtop), W // 2,
                         _native.ptr_array([row(o, r0) for o in out]), W, len(ms), r1 - r0, W,
                         s))
        torch.cuda.synchronize()
        del top, bot


def test_c4_65536_strips_seams_and_offsets_past_2_31():
    lib = _native.load()
    N, P = 65536, 8
    pan = torch.empty((N, N), device="cuda")
    synth.device_plane(pan, SEED, synth.plane_id(0, -1))
    ms = torch.empty((N // 2, N // 2), device="cuda")
    synth.device_plane(ms, SEED, synth.plane_id(0, 0))
    whole = wf.fuse(pan, [ms], wf.DwtReplace(wf.WaveletKind.DAUB4))[0]
    cuts = [k * N // P for k in range(P + 1)]
    strips = torch.empty_like(pan)
    _strips(lib.wf_fuse_strip_f32, pan, [ms], [strips], cuts)
    assert torch.equal(strips, whole)
    del strips
    exact = torch.empty_like(pan)
    _strips(lib.wf_fuse_strip_exact_f32, pan, [ms], [exact], cuts)

    def pf(rows, cols):
        return synth.hash_plane(SEED, synth.plane_id(0, -1), rows % N, cols % N)

    def bf(rows, cols):
        return synth.hash_plane(SEED, synth.plane_id(0, 0), rows % (N // 2), cols % (N // 2))

    wins = [(0, 4, 0, 64), (0, 4, N - 64, N), (N - 4, N, 0, 64), (N - 4, N, N - 64, N),
            (40000, 40004, 1000, 1128),            # element offsets > 2^31
            (N - 2, N, N // 2 - 32, N // 2 + 32)]
    for c in cuts[1:-1]:                            # every strip seam, both sides
        wins += [(c - 4, c + 4, 0, 64), (c - 4, c + 4, N - 96, N)]
    assert any(r0 * N > 2 ** 31 for r0, _, _, _ in wins)  # 32-bit offsets would wrap
    worst = 0.0
    for r0, r1, c0, c1 in wins:
        ref = O.fuse_window(pf, [bf], "daub4", r0, r1, c0, c1)[0]
        got = whole[r0:r1, c0:c1].cpu().numpy().astype(np.float64)
        worst = max(worst, float(np.abs(got - ref).max()))
        assert np.array_equal(exact[r0:r1, c0:c1].cpu().numpy(), ref.astype(np.float32)), \
            (r0, c0)
    assert worst <= 1e-3, worst
    print(f"C4 65536^2: strips == whole; windows worst max-abs {worst:.2e}; exact strips "
          "bit-identical to the oracle")


@pytest.mark.parametrize("kname", ["haar", "daub4"])
def test_landsat_qnr_scene_kernel_vs_float64_and_oracle(kname, monkeypatch):
    kind = wf.WaveletKind.HAAR if kname == "haar" else wf.WaveletKind.DAUB4
    H, W, B = 14000, 16000, 6
    pan = torch.empty((H, W), device="cuda")
    synth.device_plane(pan, SEED, synth.plane_id(0, -1))
    ms = []
    for b in range(B):
        t = torch.empty((H // 2, W // 2), device="cuda")
        synth.device_plane(t, SEED, synth.plane_id(0, b))
        ms.append(t)
    fused = wf.fuse(pan, ms, wf.DwtReplace(kind))
    fast = wf.qnr(fused, ms, pan)
    monkeypatch.setenv("WF_QNR_PATH", "generic")
    slow = wf.qnr(fused, ms, pan)
    for f in ("ergas", "d_lambda", "d_s", "qnr"):
        assert abs(getattr(fast, f) - getattr(slow, f)) <= 1e-6, (f, getattr(fast, f),
                                                                   getattr(slow, f))
    assert np.allclose(fast.q_per_band, slow.q_per_band, rtol=0, atol=1e-6)
    monkeypatch.delenv("WF_QNR_PATH")
    # a 2048 x 2048 crop (1024 x 1024 MS) against the oracle
    c = 2048
    crop_f = [f[:c, :c].contiguous() for f in fused]
    crop_m = [m[:c // 2, :c // 2].contiguous() for m in ms]
    crop_p = pan[:c, :c].contiguous()
    got = wf.qnr(crop_f, crop_m, crop_p)
    ref = Q.qnr([f.cpu().numpy() for f in crop_f], [m.cpu().numpy() for m in crop_m],
                crop_p.cpu().numpy())
    for f in ("ergas", "d_lambda", "d_s", "qnr"):
        assert abs(getattr(got, f) - ref[f]) <= 1e-6, (f, getattr(got, f), ref[f])
    assert np.allclose(got.q_per_band, ref["q_per_band"], rtol=0, atol=1e-6)
