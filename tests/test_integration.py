"""Host-side integration with the installed reference (baseline/_ref, staged by
tools/stage_reference_suite.sh): integration.install() rebinds every binding
site SURVEY.md 8(b) lists and uninstall() restores the reference; split /
merge (reference tiling.py:93-152) move tiles exactly like the reference's.
No GPU compute here (data movement and rebinding only)."""

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1803_00737_b200 as wf

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "wavefuse").is_dir():
        pytest.skip("reference not installed in baseline/_ref (tools/stage_reference_suite.sh)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import wavefuse

    return wavefuse


def test_install_rebinds_and_uninstall_restores(ref):
    import wavefuse.cluster as Cl
    import wavefuse.fusion as F
    import wavefuse.metrics as M
    import wavefuse.tiling as T

    from paper_1803_00737_b200 import integration

    before = (F.fuse_dwt, F.dwt2d_forward, M.qnr, M.resample_bilinear, T.fuse_tiled,
              Cl.WorkerServer.handle_task, ref.fuse_dwt)
    h = integration.install()
    try:
        assert integration.install() is h  # idempotent
        after = (F.fuse_dwt, F.dwt2d_forward, M.qnr, M.resample_bilinear, T.fuse_tiled,
                 Cl.WorkerServer.handle_task, ref.fuse_dwt)
        assert all(a is not b for a, b in zip(after, before))
        assert F.fuse_dwt.__wrapped__ is wf.fuse_dwt
        assert M.qnr.__wrapped__ is wf.qnr
    finally:
        h.uninstall()
    restored = (F.fuse_dwt, F.dwt2d_forward, M.qnr, M.resample_bilinear, T.fuse_tiled,
                Cl.WorkerServer.handle_task, ref.fuse_dwt)
    assert all(a is b for a, b in zip(restored, before))


@pytest.mark.parametrize("gw,gh", [(1, 1), (2, 3), (4, 2)])
def test_split_merge_match_reference(ref, gw, gh):
    import wavefuse.tiling as T

    rng = np.random.default_rng(gw * 10 + gh)
    h, w = 12 * gh, 8 * gw
    pan = rng.uniform(0, 255, (h, w)).astype(np.float32)
    ms = [rng.uniform(0, 255, (h // 2, w // 2)) for _ in range(3)]
    g_ref, g = T.plan_grid(w, h, gw, gh), wf.plan_grid(w, h, gw, gh)
    want, got = T.split(pan, ms, g_ref), wf.split(pan, ms, g)
    assert len(want) == len(got)
    for a, b in zip(want, got):
        assert a.index == b.index
        assert np.array_equal(a.pan, b.pan) and a.pan.dtype == b.pan.dtype
        assert all(np.array_equal(x, y) for x, y in zip(a.ms, b.ms))
        assert b.pan.flags.c_contiguous
    bands = [[t.pan, t.pan * 2] for t in got]
    for x, y in zip(T.merge(bands, g_ref), wf.merge(bands, g)):
        assert np.array_equal(x, y)


def test_split_merge_errors(ref):
    g = wf.plan_grid(8, 8, 2, 2)
    with pytest.raises(wf.DimensionMismatch):
        wf.split(np.zeros((8, 6)), [], g)
    with pytest.raises(wf.DimensionMismatch):
        wf.split(np.zeros((8, 8)), [np.zeros((4, 3))], g)
    with pytest.raises(wf.MissingTile):
        wf.merge([[np.zeros((4, 4))]] * 3, g)
    with pytest.raises(wf.MissingTile):
        wf.merge([[np.zeros((4, 4))]] * 3 + [None], g)
    with pytest.raises(wf.DimensionMismatch):
        wf.merge([[np.zeros((4, 4))]] * 3 + [[np.zeros((4, 2))]], g)
