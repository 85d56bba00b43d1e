"""Pin the CPU oracle (oracle/) before trusting it as the GPU checker.

1. Against golden vectors produced by the reference itself
   (tests/golden/make_golden.py imports /root/reference/pkg/src/wavefuse):
   bit-exact for transforms, resample and fusion; metrics to 1e-12.
2. Against the reference's own known-answer and property tests, restated
   (file:line of each reference test cited).
3. The closed forms the CUDA kernels implement and the
   windowed-oracle property (F4) used for scenes too big for the host.
"""

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import cpu_dwt as O
from oracle import cpu_quality as Q

KINDS = ("haar", "daub4")


def _cases(g):
    return sorted({k.split("/")[0] for k in g.keys() if k.endswith("/pan")})


# ---------------------------------------------------------------- golden ---
def test_fusion_matches_reference_golden(golden_fusion):
    g = golden_fusion
    for name in _cases(g):
        pan = g[f"{name}/pan"]
        nb = sum(1 for k in g.keys() if k.startswith(f"{name}/ms"))
        bands = [g[f"{name}/ms{b}"] for b in range(nb)]
        for kind in KINDS:
            if f"{name}/{kind}/out0" not in g:
                continue
            outs = O.fuse(pan, bands, kind)
            for b, o in enumerate(outs):
                ref = g[f"{name}/{kind}/out{b}"]
                assert o.dtype == ref.dtype, (name, kind)
                assert np.array_equal(o, ref), (name, kind, b)


def test_transforms_match_reference_golden(golden_transforms):
    g = golden_transforms
    for key in g.keys():
        if key.endswith("/fwd") or key.endswith("/inv"):
            tag, kind, op = key.rsplit("/", 2)
            if tag.startswith("v"):
                x = g[f"{tag}/x"]
                got = O.dwt1d_forward(x, kind) if op == "fwd" else O.dwt1d_inverse(x, kind)
            else:
                src = g[f"{tag}/x"] if op == "fwd" else g[f"{tag}/c"]
                got = O.dwt2d_forward(src, kind) if op == "fwd" else O.dwt2d_inverse(src, kind)
            ref = g[key]
            assert got.dtype == ref.dtype
            assert np.array_equal(got, ref), key
        elif key.endswith("/out") and key.startswith("rs"):
            tag = key[: -len("/out")]
            x = g[f"{tag}/x"]
            ref = g[key]
            got = O.resample_bilinear(x, ref.shape[1], ref.shape[0])
            assert got.dtype == ref.dtype
            assert np.array_equal(got, ref), key


def test_metrics_match_reference_golden(golden_metrics):
    g = golden_metrics
    for k in range(5):
        assert abs(Q.q_index(g[f"q{k}/a"], g[f"q{k}/b"]) - float(g[f"q{k}/q"])) <= 1e-12
    assert Q.q_index(g["qdeg/a"], g["qdeg/b"]) == float(g["qdeg/q"])
    for k in range(4):
        tag = f"rep{k}"
        nb = sum(1 for key in g.keys() if key.startswith(f"{tag}/ms"))
        ms = [g[f"{tag}/ms{b}"] for b in range(nb)]
        fused = [g[f"{tag}/fused{b}"] for b in range(nb)]
        rep = Q.qnr(fused, ms, g[f"{tag}/pan"])
        assert abs(rep["ergas"] - float(g[f"{tag}/ergas"])) <= 1e-12
        assert np.allclose(rep["q_per_band"], g[f"{tag}/q_per_band"], rtol=0, atol=1e-12)
        assert abs(rep["d_lambda"] - float(g[f"{tag}/d_lambda"])) <= 1e-12
        assert abs(rep["d_s"] - float(g[f"{tag}/d_s"])) <= 1e-12
        assert abs(rep["qnr"] - float(g[f"{tag}/qnr"])) <= 1e-12
        assert np.array_equal(Q.degrade(fused[0], 2), g[f"{tag}/degrade0"])


# ------------------------------------------- reference known answers -----
def test_filter_taps():
    """test_wavelet.py:34-53"""
    h, g, even, odd = O.taps()
    s3, sc = math.sqrt(3.0), 4.0 * math.sqrt(2.0)
    assert np.allclose(h, [(1 + s3) / sc, (3 + s3) / sc, (3 - s3) / sc, (1 - s3) / sc],
                       atol=1e-12, rtol=0)
    assert abs(sum(h) - math.sqrt(2.0)) < 1e-12 and abs(sum(g)) < 1e-12
    assert abs(h[0] - 0.4829629131) < 1e-9 and abs(h[3] + 0.1294095226) < 1e-9
    assert even == [h[2], g[2], h[0], g[0]] and odd == [h[3], g[3], h[1], g[1]]


def test_haar_known_answers():
    """test_wavelet.py:62-74, 143-154"""
    assert np.allclose(O.dwt1d_forward(np.array([6.0, 2.0, 4.0, 8.0]), "haar"), [4, 6, 2, -2])
    assert np.allclose(O.dwt1d_inverse(np.array([4.0, 6.0, 2.0, -2.0]), "haar"), [6, 2, 4, 8])
    out = O.dwt2d_forward(np.array([[1.0, 3.0], [5.0, 7.0]]), "haar")
    assert np.allclose(out, [[4.0, -1.0], [-2.0, 0.0]], atol=1e-12)
    back = O.dwt2d_inverse(np.array([[4.0, -1.0], [-2.0, 0.0]]), "haar")
    assert np.allclose(back, [[1.0, 3.0], [5.0, 7.0]], atol=1e-12)


def test_d4_constant_and_dense_matrix():
    """test_wavelet.py:21-31, 77-93"""
    assert np.allclose(O.dwt1d_forward(np.ones(8), "daub4"), [math.sqrt(2.0)] * 4 + [0.0] * 4,
                       atol=1e-6)
    h, g, _, _ = O.taps()
    rng = np.random.default_rng(42)
    for n in (4, 8, 16):
        m = np.zeros((n, n))
        for i in range(n // 2):
            for k in range(4):
                m[i, (2 * i + k) % n] += h[k]
                m[n // 2 + i, (2 * i + k) % n] += g[k]
        for _ in range(5):
            x = rng.uniform(0.0, 255.0, n)
            assert np.allclose(O.dwt1d_forward(x, "daub4"), m @ x, atol=1e-9)
            c = rng.uniform(-255.0, 255.0, n)
            assert np.allclose(O.dwt1d_inverse(c, "daub4"), np.linalg.solve(m, c), atol=1e-9)


@pytest.mark.parametrize("kind", KINDS)
def test_perfect_reconstruction(kind):
    """test_wavelet.py:167-188; test_acceptance.py:69-86"""
    rng = np.random.default_rng(6)
    for shape in ((4, 4), (6, 10), (64, 64)):
        p = rng.uniform(0.0, 255.0, shape)
        assert np.max(np.abs(O.dwt2d_inverse(O.dwt2d_forward(p, kind), kind) - p)) <= 1e-9
        p32 = p.astype(np.float32)
        b32 = O.dwt2d_inverse(O.dwt2d_forward(p32, kind), kind)
        assert b32.dtype == np.float32
        assert np.max(np.abs(b32.astype(np.float64) - p32)) <= 1e-4


def test_fusion_known_answers():
    """test_fusion.py:127-158"""
    assert np.allclose(O.fuse_dwt(np.full((4, 4), 100.0), np.full((2, 2), 50.0), "haar"), 50.0)
    assert np.allclose(O.fuse_dwt(np.full((8, 8), 100.0), np.full((4, 4), 50.0), "daub4"), 50.0)
    out = O.fuse_dwt(np.array([[1.0, 3.0], [5.0, 7.0]]), np.array([[10.0]]), "haar")
    assert np.allclose(out, [[7.0, 9.0], [11.0, 13.0]], atol=1e-9)
    rng = np.random.default_rng(13)
    for kind, gain in (("haar", 1.0), ("daub4", 2.0)):
        pan = rng.uniform(0, 255, (16, 16))
        ms = O.dwt2d_forward(pan, kind)[:8, :8] / gain
        assert np.max(np.abs(O.fuse_dwt(pan, ms, kind) - pan)) < 1e-4


def test_metric_known_answers():
    """test_metrics.py:14-99"""
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert abs(Q.q_index(a, 2.0 * a) - 0.64) < 1e-12
    assert Q.q_index(np.full((4, 4), 5.0), np.full((4, 4), 5.0)) == 1.0
    assert Q.q_index(np.full((4, 4), 5.0), np.full((4, 4), 7.0)) == 0.0
    z = np.array([[-1.0, 1.0], [-1.0, 1.0]])
    assert Q.q_index(z, -z) == 0.0
    assert abs(Q.ergas([np.full((16, 16), 105.0)], [np.full((8, 8), 100.0)], 2) - 2.5) < 1e-12
    rng = np.random.default_rng(24)
    ref = [rng.uniform(1, 255, (8, 8)) for _ in range(3)]
    assert Q.ergas([np.kron(r, np.ones((2, 2))) for r in ref], ref, 2) == 0.0


# --------------------------------------------- closed forms the kernels use
def closed_form(pan, band, kind):
    """SURVEY.md F1/F2 in float64: Haar out = pan + (ms - mean2x2(pan));
    D4 out = pan + S_LL(2 ms - LL(pan)), periodic."""
    p = np.asarray(pan, dtype=np.float64)
    m = np.asarray(band, dtype=np.float64)
    if kind == "haar":
        ll = 0.25 * (p[0::2, 0::2] + p[0::2, 1::2] + p[1::2, 0::2] + p[1::2, 1::2])
        return p + np.kron(m - ll, np.ones((2, 2)))
    h, _, _, _ = O.taps()
    H, W = p.shape
    r = np.arange(H // 2) * 2
    c = np.arange(W // 2) * 2
    rows = sum(h[k] * p[(r + k) % H] for k in range(4))          # (H/2, W)
    ll = sum(h[l] * rows[:, (c + l) % W] for l in range(4))       # (H/2, W/2)
    e = 2.0 * m - ll
    ep = np.roll(e, 1, axis=0)
    v = np.empty((H, W // 2))
    v[0::2] = h[2] * ep + h[0] * e
    v[1::2] = h[3] * ep + h[1] * e
    vp = np.roll(v, 1, axis=1)
    s = np.empty((H, W))
    s[:, 0::2] = h[2] * vp + h[0] * v
    s[:, 1::2] = h[3] * vp + h[1] * v
    return p + s


@pytest.mark.parametrize("kind", KINDS)
def test_closed_form_equals_transform_path(kind):
    rng = np.random.default_rng(5)
    for h, w in ((4, 4), (8, 12), (34, 70), (64, 130)):
        pan = rng.uniform(0, 255, (h, w))
        band = rng.uniform(0, 255, (h // 2, w // 2))
        assert np.max(np.abs(closed_form(pan, band, kind) - O.fuse_dwt(pan, band, kind))) < 1e-10


@pytest.mark.parametrize("kind", KINDS)
def test_windowed_oracle_is_exact(kind):
    """a window fused with a wrapped 4-px margin equals the
    global result bit for bit, including windows that wrap the edges."""
    rng = np.random.default_rng(8)
    H, W = 64, 96
    pan = rng.uniform(0, 255, (H, W)).astype(np.float32)
    bands = [rng.uniform(0, 255, (H // 2, W // 2)).astype(np.float32) for _ in range(2)]
    full = O.fuse(pan, bands, kind)

    def pf(rows, cols):
        return O.wrapped_window(pan, rows[0], rows[-1] + 1, cols[0], cols[-1] + 1)

    def bf(b):
        return lambda rows, cols: O.wrapped_window(b, rows[0], rows[-1] + 1, cols[0], cols[-1] + 1)

    for r0, r1, c0, c1 in ((0, 16, 0, 32), (48, 64, 80, 96), (20, 40, 10, 50), (0, 64, 0, 96)):
        win = O.fuse_window(pf, [bf(b) for b in bands], kind, r0, r1, c0, c1)
        for wv, fv in zip(win, full):
            assert np.array_equal(wv, fv[r0:r1, c0:c1])


@pytest.mark.parametrize("kind", KINDS)
def test_parallel_cpu_baseline_is_exact(kind):
    rng = np.random.default_rng(9)
    pan = rng.uniform(0, 255, (200, 64)).astype(np.float32)
    bands = [rng.uniform(0, 255, (100, 32)).astype(np.float32) for _ in range(3)]
    ref = O.fuse(pan, bands, kind)
    got = O.fuse_parallel(pan, bands, kind, threads=3, strip_rows=48)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_quantized_path_matches_reference_golden():
    """8 bpp worker computation (tiling.py:163-172, 268-269) and quantize
    (imageio.py:115-123), bit-exact against the reference's outputs."""
    g = np.load(Path(__file__).parent / "golden" / "quantized.npz")
    assert np.array_equal(O.quantize(g["quantize/in"]), g["quantize/out"])
    for k in range(4):
        nb = sum(1 for key in g.files if key.startswith(f"t{k}/ms"))
        pan = g[f"t{k}/pan"]
        ms = [g[f"t{k}/ms{b}"] for b in range(nb)]
        for kind in KINDS:
            got = O.fuse_quantized(pan, ms, kind)
            for b, o in enumerate(got):
                assert np.array_equal(o, g[f"t{k}/{kind}/out{b}"]), (k, kind, b)


# --- PNM front end (oracle/cpu_raster.py) against the reference CLI's files ---

from oracle import cpu_raster as R  # noqa: E402

PNM_CASES = ("rgb", "gray2", "gray1", "rs")


def _pnm_inputs(g, name):
    ms = [g[k].tobytes() for k in sorted(k for k in g.keys() if k.startswith(f"{name}/ms"))]
    return g[f"{name}/pan"].tobytes(), ms, [int(v) for v in g[f"{name}/grid"]]


@pytest.mark.parametrize("name", PNM_CASES)
@pytest.mark.parametrize("method,kind", [("hdwt", "haar"), ("ddwt", "daub4")])
def test_cli_fuse_oracle_matches_reference_files(golden_pnm, name, method, kind):
    pan, ms, (gw, gh) = _pnm_inputs(golden_pnm, name)
    got = R.cli_fuse(pan, ms, kind, gw, gh)
    want = [golden_pnm[k].tobytes() for k in sorted(
        k for k in golden_pnm.keys() if k.startswith(f"{name}/{method}/out"))]
    assert got == want


def test_pad_oracle_matches_reference(golden_pnm):
    for name in ("p0", "p1", "p2"):
        src, want = golden_pnm[f"pad/{name}/in"], golden_pnm[f"pad/{name}/out"]
        got = R.pad_edge(src, want.shape[1], want.shape[0])
        assert got.dtype == want.dtype and np.array_equal(got, want)
    pan, ms = golden_pnm["padin/pan"], [golden_pnm["padin/ms0"], golden_pnm["padin/ms1"]]
    pp, mp = R.pad_inputs(pan, ms, 4, 3)
    assert np.array_equal(pp, golden_pnm["padin/out_pan"])
    assert np.array_equal(mp[0], golden_pnm["padin/out_ms0"])
    assert np.array_equal(mp[1], golden_pnm["padin/out_ms1"])
