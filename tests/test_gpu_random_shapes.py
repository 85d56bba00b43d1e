"""Randomised shapes through every fusion path against the pinned oracle:
the fast kernels within the north star's 1e-3 (measured <= 2e-4 for f32,
~1e-12 for f64), the exact kernels bit for bit, the 8 bpp kernels within one
LSB (Haar bit-exact), for widths that exercise the TMA, register and scalar
variants (W % 32, W % 16, W % 4, W = 2 mod 4), heights from the minimum up,
and 1..9 bands (several launches past 8)."""
import numpy as np
import pytest
import torch

import paper_1803_00737_b200 as wf
from oracle import cpu_dwt as O

pytestmark = pytest.mark.gpu

KINDS = {"haar": wf.WaveletKind.HAAR, "daub4": wf.WaveletKind.DAUB4}


def _shapes(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        h = int(rng.choice([4, 6, 8, 18, 34, 66, 130]))
        w = int(rng.choice([4, 6, 10, 32, 34, 64, 96, 130, 258, 544, 1090]))
        nb = int(rng.integers(1, 10))
        out.append((h, w, nb))
    return out


@pytest.mark.parametrize("kname", list(KINDS))
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_fast_and_exact_random_shapes(kname, dt):
    rng = np.random.default_rng(100 + len(kname) + (dt == np.float64))
    tol = 1e-3 if dt == np.float32 else 1e-9
    for h, w, nb in _shapes(7 + (dt == np.float64), 12):
        pan = rng.uniform(0, 255, (h, w)).astype(dt)
        bands = [rng.uniform(0, 255, (h // 2, w // 2)).astype(dt) for _ in range(nb)]
        ref = O.fuse(pan, bands, kname)
        m = wf.DwtReplace(KINDS[kname])
        fast_h = wf.fuse(pan, bands, m)
        fast_d = wf.fuse(torch.from_numpy(pan).cuda(), [torch.from_numpy(b).cuda() for b in bands],
                         m)
        exact = wf.fuse(pan, bands, m, exact=True)
        for r, a, b, e in zip(ref, fast_h, fast_d, exact):
            assert np.max(np.abs(a.astype(np.float64) - r)) <= tol, (h, w, nb)
            assert np.array_equal(a, b.cpu().numpy()), (h, w, nb)
            assert np.array_equal(e, r), (h, w, nb)


@pytest.mark.parametrize("kname", list(KINDS))
def test_u8_random_shapes(kname):
    rng = np.random.default_rng(300 + len(kname))
    for h, w, nb in _shapes(11, 10):
        pan = rng.integers(0, 256, (h, w), dtype=np.uint8)
        bands = [rng.integers(0, 256, (h // 2, w // 2), dtype=np.uint8) for _ in range(nb)]
        ref = O.fuse_quantized(pan, bands, kname)
        got = wf.fuse_quantized(pan, bands, wf.DwtReplace(KINDS[kname]))
        exact = wf.fuse_quantized(pan, bands, wf.DwtReplace(KINDS[kname]), exact=True)
        for r, g, e in zip(ref, got, exact):
            d = np.abs(g.astype(np.int32) - r.astype(np.int32))
            assert d.max() <= (0 if kname == "haar" else 1), (h, w, nb)
            assert np.array_equal(e, r), (h, w, nb)


@pytest.mark.parametrize("kname", list(KINDS))
def test_fuse_and_qnr_random_shapes(kname):
    """fuse_and_qnr on random shapes and band counts (the one-call fuse +
    report where the scene qualifies, fuse() + qnr() where it does not:
    W % 8 != 0, H or W < 64, one band): fused bands as fuse() (float32 within
    the north star's 1e-3 of the oracle) and the report within 1e-6 of the
    pinned oracle's qnr() of those bands, device and numpy inputs."""
    from oracle import cpu_quality as Q

    rng = np.random.default_rng(500 + len(kname))
    shapes = [(64, 64, 2), (96, 136, 3), (128, 200, 6), (160, 264, 8), (66, 130, 4),
              (256, 96, 5), (34, 70, 2)]
    m = wf.DwtReplace(KINDS[kname])
    for h, w, nb in shapes:
        pan = rng.uniform(0, 255, (h, w)).astype(np.float32)
        bands = [rng.uniform(1, 255, (h // 2, w // 2)).astype(np.float32) for _ in range(nb)]
        f_dev, rep_dev = wf.fuse_and_qnr(torch.from_numpy(pan).cuda(),
                                         [torch.from_numpy(b).cuda() for b in bands], m)
        f_np, rep_np = wf.fuse_and_qnr(pan, bands, m)
        fused = [f.cpu().numpy() for f in f_dev]
        for a, b, r in zip(fused, f_np, O.fuse(pan, bands, kname)):
            assert np.array_equal(a, b), (h, w, nb)
            assert np.max(np.abs(a.astype(np.float64) - r)) <= 1e-3, (h, w, nb)
        ref = Q.qnr(fused, bands, pan)
        for rep in (rep_dev, rep_np):
            assert abs(rep.ergas - ref["ergas"]) <= 1e-6, (h, w, nb)
            assert abs(rep.qnr - ref["qnr"]) <= 1e-6, (h, w, nb)
            assert abs(rep.d_lambda - ref["d_lambda"]) <= 1e-6, (h, w, nb)
            assert abs(rep.d_s - ref["d_s"]) <= 1e-6, (h, w, nb)
            assert np.allclose(rep.q_per_band, ref["q_per_band"], rtol=0, atol=1e-6), (h, w, nb)
