"""Fusion quality metrics on the GPU: degrade, Q-index, ERGAS, D_lambda, D_s,
QNR.

Drop-in for /root/reference/pkg/src/wavefuse/metrics.py (same names,
signatures, validation order and exception classes). All statistics are
float64 on the device (csrc/quality.cu): two-pass block moments per 32x32 Q
block with the reference's degenerate rule, deterministic reductions. Planes
may be numpy arrays or CUDA tensors (float32 planes are read as float32 and
widened exactly in-kernel, so no float64 copy of a fused scene is made).
Scalars come back to the host once per public call.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .errors import DimensionMismatch, NotDivisible, TooFewBands, ZeroBandMean

BLOCK = 32  # metrics.py:17


@dataclass(frozen=True)
class QualityReport:
    """metrics.py:20-28"""

    ergas: float
    q_per_band: list[float]
    d_lambda: float
    d_s: float
    qnr: float


# ---------------------------------------------------------------- plumbing --
def _shape(x):
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def _plane(x) -> torch.Tensor:
    """Contiguous CUDA tensor, float32 kept as float32, everything else
    float64 (the reference casts everything to float64, metrics.py:86-91;
    float32 -> float64 is exact and happens in-kernel)."""
    dt = np.float32 if _device.is_f32(x) else np.float64
    return _device.to_device(x, dt)


def _is64(t: torch.Tensor) -> int:
    return 1 if t.dtype == torch.float64 else 0


def _bands(image) -> list:
    """metrics.py:86-91: list of planes, all the same shape."""
    bands = [b if isinstance(b, torch.Tensor) else np.asarray(b) for b in image]
    for b in bands[1:]:
        if _shape(b) != _shape(bands[0]):
            raise DimensionMismatch(f"band sizes differ: {_shape(b)} vs {_shape(bands[0])}")
    return bands


class _Results:
    """A device float64 vector the kernels write scalars into; read once."""

    def __init__(self, n: int, device):
        self.t = torch.zeros(max(1, n), dtype=torch.float64, device=device)
        self.n = 0

    def slot(self) -> int:
        self.n += 1
        return self.n - 1

    def host(self) -> np.ndarray:
        return self.t.cpu().numpy()


def _q_into(res: _Results, a: torch.Tensor, b: torch.Tensor) -> int:
    h, w = a.shape
    lib = _native.load()
    ws = torch.empty(int(lib.wf_q_index_workspace_bytes(h, w)) // 8 + 1, dtype=torch.float64,
                     device=a.device)
    idx = res.slot()
    _native.check(lib.wf_q_index(a.data_ptr(), _is64(a), a.stride(0), b.data_ptr(), _is64(b),
                                 b.stride(0), h, w, ws.data_ptr(), res.t.data_ptr(), idx,
                                 _device.stream_ptr()))
    return idx


def _degrade_dev(p: torch.Tensor, factor: int) -> torch.Tensor:
    h, w = p.shape
    out = torch.empty((h // factor, w // factor), dtype=torch.float64, device=p.device)
    _native.check(_native.load().wf_degrade(p.data_ptr(), _is64(p), p.stride(0), h, w, factor,
                                            out.data_ptr(), out.stride(0), _device.stream_ptr()))
    return out


def _upsample_dev(b: torch.Tensor, w: int, h: int) -> torch.Tensor:
    """metrics.py:122-123 on a float64-cast band: bit-identical to the
    reference's resample_bilinear(band.astype(float64), w, h)."""
    if tuple(b.shape) == (h, w):
        return b
    lib = _native.load()
    out = torch.empty((h, w), dtype=torch.float64, device=b.device)
    bh, bw = b.shape
    fn = lib.wf_resample_bilinear_f64 if b.dtype == torch.float64 else lib.wf_resample_bilinear_f32_to_f64
    _native.check(fn(b.data_ptr(), b.stride(0), bh, bw, out.data_ptr(), w, h, w,
                     _device.stream_ptr()))
    return out


# ------------------------------------------------------------ public API ---
def degrade(plane, factor: int):
    """metrics.py:31-42: factor x factor block mean, float64."""
    if factor < 1:
        raise ValueError(f"factor {factor} must be >= 1")
    shape = _shape(plane)
    if factor == 1:
        if isinstance(plane, torch.Tensor):
            return plane.to(torch.float64).clone()
        return np.array(plane, dtype=np.float64, copy=True)
    h, w = shape
    if h % factor or w % factor:
        raise NotDivisible(f"{w}x{h} not divisible by {factor}")
    out = _degrade_dev(_plane(plane), factor)
    return out if isinstance(plane, torch.Tensor) else _device.to_host(out)


def q_index(a, b) -> float:
    """metrics.py:57-83: block-averaged universal image quality index."""
    if _shape(a) != _shape(b):
        raise DimensionMismatch(f"planes differ: {_shape(a)} vs {_shape(b)}")
    ta, tb = _plane(a), _plane(b)
    res = _Results(1, ta.device)
    _q_into(res, ta, tb)
    return float(res.host()[0])


def _ergas_checks(f_bands, r_bands, ratio):
    if ratio < 1:
        raise ValueError(f"ratio {ratio} must be >= 1")
    if len(f_bands) != len(r_bands):
        raise DimensionMismatch(f"band counts differ: {len(f_bands)} vs {len(r_bands)}")
    rh, rw = _shape(r_bands[0])
    if _shape(f_bands[0]) != (rh * ratio, rw * ratio):
        raise DimensionMismatch(
            f"fused {_shape(f_bands[0])} is not reference {_shape(r_bands[0])} times {ratio}"
        )


def _ergas_into(res: _Results, f_t, r_t, ratio) -> list[int]:
    lib = _native.load()
    rh, rw = r_t[0].shape
    ws = torch.empty(int(lib.wf_ergas_workspace_bytes(rh, rw)) // 8 + 1, dtype=torch.float64,
                     device=r_t[0].device)
    slots = []
    for fb, rb in zip(f_t, r_t):
        i0 = res.slot()
        res.slot()
        _native.check(lib.wf_ergas_band(fb.data_ptr(), _is64(fb), fb.stride(0), rb.data_ptr(),
                                        _is64(rb), rb.stride(0), rh, rw, ratio, ws.data_ptr(),
                                        res.t.data_ptr() + 8 * i0, _device.stream_ptr()))
        slots.append(i0)
    return slots


def _ergas_value(vals: np.ndarray, slots: list[int], ratio: int) -> float:
    acc = 0.0
    for i0 in slots:
        mse, mu = float(vals[i0]), float(vals[i0 + 1])
        if mu == 0.0:
            raise ZeroBandMean("reference band mean is zero")
        acc += mse / (mu * mu)
    return 100.0 / ratio * float(np.sqrt(acc / len(slots)))


def ergas(fused, ms_ref, ratio: int) -> float:
    """metrics.py:94-119"""
    if ratio < 1:
        raise ValueError(f"ratio {ratio} must be >= 1")
    f_bands, r_bands = _bands(fused), _bands(ms_ref)
    _ergas_checks(f_bands, r_bands, ratio)
    f_t = [_plane(b) for b in f_bands]
    r_t = [_plane(b) for b in r_bands]
    res = _Results(2 * len(f_t), f_t[0].device)
    slots = _ergas_into(res, f_t, r_t, ratio)
    return _ergas_value(res.host(), slots, ratio)


def _dlambda_checks(f_bands, m_bands):
    n = len(f_bands)
    if n != len(m_bands):
        raise DimensionMismatch(f"band counts differ: {n} vs {len(m_bands)}")
    if n < 2:
        raise TooFewBands("inter-band comparison needs at least 2 bands")


def _dlambda_into(res, f_t, up_t) -> list[tuple[int, int]]:
    n = len(f_t)
    return [(_q_into(res, f_t[k], f_t[l]), _q_into(res, up_t[k], up_t[l]))
            for k in range(n) for l in range(k + 1, n)]


def _dlambda_value(vals, pairs, n) -> float:
    total = 0.0
    for i, j in pairs:
        total += 2.0 * abs(float(vals[i]) - float(vals[j]))
    return min(1.0, max(0.0, total / (n * (n - 1))))


def d_lambda(fused, ms) -> float:
    """metrics.py:126-142: spectral distortion."""
    f_bands, m_bands = _bands(fused), _bands(ms)
    _dlambda_checks(f_bands, m_bands)
    f_t = [_plane(b) for b in f_bands]
    fh, fw = f_t[0].shape
    up_t = [_upsample_dev(_plane(b), fw, fh) for b in m_bands]
    n = len(f_t)
    res = _Results(n * (n - 1), f_t[0].device)
    pairs = _dlambda_into(res, f_t, up_t)
    return _dlambda_value(res.host(), pairs, n)


def _infer_ratio(pan_shape, ms_shape) -> int:
    """metrics.py:145-152"""
    ph, pw = pan_shape
    mh, mw = ms_shape
    if mh == 0 or mw == 0 or ph % mh or pw % mw or ph // mh != pw // mw:
        raise DimensionMismatch(
            f"panchromatic {tuple(pan_shape)} is not an integer multiple of bands {tuple(ms_shape)}"
        )
    return ph // mh


def _ds_checks(f_bands, m_bands, pan) -> int:
    if len(f_bands) != len(m_bands):
        raise DimensionMismatch(f"band counts differ: {len(f_bands)} vs {len(m_bands)}")
    if _shape(f_bands[0]) != _shape(pan):
        raise DimensionMismatch(
            f"fused {_shape(f_bands[0])} does not match panchromatic {_shape(pan)}"
        )
    return _infer_ratio(_shape(pan), _shape(m_bands[0]))


def _ds_into(res, f_t, m_t, p_t, ratio):
    low = _degrade_dev(p_t, ratio) if ratio != 1 else p_t
    return [(_q_into(res, fb, p_t), _q_into(res, mb, low)) for fb, mb in zip(f_t, m_t)]


def _ds_value(vals, pairs) -> float:
    total = sum(abs(float(vals[i]) - float(vals[j])) for i, j in pairs)
    return min(1.0, max(0.0, total / len(pairs)))


def d_s(fused, ms, pan) -> float:
    """metrics.py:155-175: spatial distortion."""
    f_bands, m_bands = _bands(fused), _bands(ms)
    ratio = _ds_checks(f_bands, m_bands, pan)
    f_t = [_plane(b) for b in f_bands]
    m_t = [_plane(b) for b in m_bands]
    p_t = _plane(pan)
    res = _Results(2 * len(f_t), p_t.device)
    pairs = _ds_into(res, f_t, m_t, p_t, ratio)
    return _ds_value(res.host(), pairs)


def _scene_launch(f_t, m_t, p_t, n, h, w, ws, out, flag) -> None:
    """wf_quality_scene_f32, or wf_quality_scene_f64 for float64 scenes."""
    lib = _native.load()
    fn = lib.wf_quality_scene_f32 if p_t.dtype == torch.float32 else lib.wf_quality_scene_f64
    _native.check(fn(
        _native.ptr_array([t.data_ptr() for t in f_t]),
        _native.ptr_array([t.data_ptr() for t in m_t]), p_t.data_ptr(), f_t[0].stride(0),
        m_t[0].stride(0), p_t.stride(0), n, h, w, ws.data_ptr(), out.data_ptr(),
        flag.data_ptr(), _device.stream_ptr()))


def _qnr_scene(f_t, m_t, p_t, ratio) -> QualityReport | None:
    """One-pass fused report (csrc/quality_scene.cu) when the scene qualifies:
    float32 or float64 planes (all one dtype), ratio 2, 2..8 bands, H, W >= 64.
    None = use the generic path (also when a block needs the element-wise
    identity test)."""
    n = len(f_t)
    h, w = p_t.shape
    if not _scene_ok((*f_t, *m_t, p_t), n, h, w, ratio):
        return None
    ws, out, flag = _scene_buffers(n, h, w, p_t.device)
    _scene_launch(f_t, m_t, p_t, n, h, w, ws, out, flag)
    if int(flag.item()):
        return None
    return _scene_report(out.cpu().numpy(), n, ratio)


def _scene_ok(tensors, n, h, w, ratio) -> bool:
    import os

    dt = tensors[-1].dtype
    if os.environ.get("WF_QNR_PATH") == "generic" or ratio != 2 or not 2 <= n <= 8 \
            or h < 64 or w < 64 or w % 8 or dt not in (torch.float32, torch.float64) \
            or any(t.dtype != dt for t in tensors) or any(t.data_ptr() % 16 for t in tensors):
        return False
    # float64: the fused bands and the PAN share one pitch (16-byte rows)
    return dt == torch.float32 or (all(t.stride(0) == tensors[-1].stride(0)
                                       for t in tensors[:n]) and tensors[-1].stride(0) % 2 == 0)


def _scene_buffers(n, h, w, device):
    lib = _native.load()
    ws = torch.empty(int(lib.wf_quality_scene_workspace_bytes(n, h, w)) // 8 + 1,
                     dtype=torch.float64, device=device)
    c = n * (n - 1) // 2
    out = torch.zeros(n + 2 * c + 4 * n, dtype=torch.float64, device=device)
    flag = torch.zeros(1, dtype=torch.int32, device=device)
    return ws, out, flag


def _scene_report(vals, n, ratio) -> QualityReport:
    """The report from the scene kernels' output vector (layout in
    include/wavefuse_b200.h, wf_quality_scene_f32)."""
    c = n * (n - 1) // 2
    fu = vals[:n]
    ff, uu = vals[n:n + c], vals[n + c:n + 2 * c]
    fp = vals[n + 2 * c:2 * n + 2 * c]
    low = vals[2 * n + 2 * c:3 * n + 2 * c]
    mse = vals[3 * n + 2 * c:4 * n + 2 * c]
    mu = vals[4 * n + 2 * c:]
    spectral = min(1.0, max(0.0, float(np.sum(2.0 * np.abs(ff - uu))) / (n * (n - 1))))
    spatial = min(1.0, max(0.0, float(np.sum(np.abs(fp - low))) / n))
    acc = 0.0
    for k in range(n):
        if mu[k] == 0.0:
            raise ZeroBandMean("reference band mean is zero")
        acc += float(mse[k]) / (float(mu[k]) * float(mu[k]))
    return QualityReport(
        ergas=100.0 / ratio * float(np.sqrt(acc / n)),
        q_per_band=[float(v) for v in fu],
        d_lambda=spectral,
        d_s=spatial,
        qnr=(1.0 - spectral) * (1.0 - spatial),
    )


class PendingReport:
    """A report whose kernels are queued on the current stream but whose
    scalars have not been read back (qnr_async). result() synchronises once
    and finishes on the host; if the scene kernel flagged a block that needs
    the element-wise identity test, result() falls back to qnr()."""

    def __init__(self, args, bufs, n, ratio):
        self._args, self._bufs, self._n, self._ratio = args, bufs, n, ratio
        self._report = None
        self._done = None
        if bufs is not None:  # result() may run on another stream than the kernels
            self._done = torch.cuda.Event()
            self._done.record(torch.cuda.current_stream())

    def result(self) -> QualityReport:
        if self._report is None:
            if self._bufs is None:
                self._report = qnr(*self._args)
            else:
                _, out, flag = self._bufs
                torch.cuda.current_stream().wait_event(self._done)
                vals = torch.cat([out, flag.to(torch.float64)]).cpu().numpy()
                if int(vals[-1]):
                    self._report = qnr(*self._args)
                else:
                    self._report = _scene_report(vals[:-1], self._n, self._ratio)
            self._bufs = None
        return self._report


def qnr_async(fused, ms, pan) -> PendingReport:
    """qnr() without the read-back: the same preconditions (raised now), the
    one-pass scene kernels queued on the current stream, the scalars read by
    PendingReport.result(). Lets a caller score many scenes back to back with
    one synchronisation (bench.py's batch workload). Scenes the one-pass
    kernel does not cover are scored by qnr() inside result()."""
    f_bands, m_bands = _bands(fused), _bands(ms)
    ratio = _infer_ratio(_shape(pan), _shape(m_bands[0]))
    _dlambda_checks(f_bands, m_bands)
    _ds_checks(f_bands, m_bands, pan)
    _ergas_checks(f_bands, m_bands, ratio)
    f_t = [_plane(b) for b in f_bands]
    m_t = [_plane(b) for b in m_bands]
    p_t = _plane(pan)
    n = len(f_t)
    h, w = p_t.shape
    if not _scene_ok((*f_t, *m_t, p_t), n, h, w, ratio):
        return PendingReport((fused, ms, pan), None, n, ratio)
    ws, out, flag = _scene_buffers(n, h, w, p_t.device)
    _scene_launch(f_t, m_t, p_t, n, h, w, ws, out, flag)
    # the workspace goes back to the caching allocator now: any later user of
    # that memory is ordered after these kernels on the same stream
    del ws
    return PendingReport((fused, ms, pan), (None, out, flag), n, ratio)


def qnr(fused, ms, pan) -> QualityReport:
    """metrics.py:178-199: the full report. All preconditions are checked
    before any compute; every Q, MSE and mean is computed on the GPU and the
    scalars are read back once. Float32 scenes at ratio 2 take the one-pass
    scene kernel; anything else the per-pair kernels."""
    f_bands, m_bands = _bands(fused), _bands(ms)
    ratio = _infer_ratio(_shape(pan), _shape(m_bands[0]))
    _dlambda_checks(f_bands, m_bands)
    _ds_checks(f_bands, m_bands, pan)
    _ergas_checks(f_bands, m_bands, ratio)
    f_t = [_plane(b) for b in f_bands]
    m_t = [_plane(b) for b in m_bands]
    p_t = _plane(pan)
    fast = _qnr_scene(f_t, m_t, p_t, ratio)
    if fast is not None:
        return fast
    fh, fw = f_t[0].shape
    up_t = [_upsample_dev(b, fw, fh) for b in m_t]
    n = len(f_t)
    res = _Results(n + n * (n - 1) + 2 * n + 2 * n, p_t.device)
    per_band = [_q_into(res, fb, ub) for fb, ub in zip(f_t, up_t)]
    dl_pairs = _dlambda_into(res, f_t, up_t)
    ds_pairs = _ds_into(res, f_t, m_t, p_t, ratio)
    e_slots = _ergas_into(res, f_t, m_t, ratio)
    vals = res.host()
    spectral = _dlambda_value(vals, dl_pairs, n)
    spatial = _ds_value(vals, ds_pairs)
    return QualityReport(
        ergas=_ergas_value(vals, e_slots, ratio),
        q_per_band=[float(vals[i]) for i in per_band],
        d_lambda=spectral,
        d_s=spatial,
        qnr=(1.0 - spectral) * (1.0 - spatial),
    )


def _fuse_quality_launch(p_t, m_t, outs, code=1):
    """Queue the fusion + report call (wf_fuse_quality_f32; code 1 = Haar, one
    pass; 2 = D4, fusion then report) of device float32 planes into `outs`
    (contiguous h x w float32) on the current stream; returns the report
    vector and the undecidable flag (not read)."""
    lib = _native.load()
    n = len(m_t)
    h, w = p_t.shape
    ws, out, flag = _scene_buffers(n, h, w, p_t.device)
    _native.check(lib.wf_fuse_quality_f32(
        code, p_t.data_ptr(), p_t.stride(0), _native.ptr_array([t.data_ptr() for t in m_t]),
        m_t[0].stride(0), _native.ptr_array([o.data_ptr() for o in outs]), w, n, h, w,
        ws.data_ptr(), out.data_ptr(), flag.data_ptr(), _device.stream_ptr()))
    return out, flag


def fuse_and_qnr_async(pan, ms, method, *, out=None):
    """fuse_and_qnr() for device tensors without the read-back: returns
    (fused, PendingReport). Float32 Haar and D4 scenes that qualify take
    wf_fuse_quality_f32 (Haar: the one-pass kernel; D4: fusion then report in
    one call), written into `out` if given (contiguous float32 h x w tensors
    on the PAN's device, one per band); anything else runs fuse() (into new
    tensors) and qnr_async(). bench.py's batch workload (C5) scores its
    scenes so."""
    from . import fusion as _fusion
    from .wavelet import WaveletKind

    if not isinstance(method, _fusion.DwtReplace):
        raise TypeError(f"unknown fusion method {method!r}")
    bands = _bands(ms)
    # (the reference-exact default, WF_EXACT=1 / set_exact_default(True),
    # fuses with the float64 kernels: fuse() then)
    if method.kind in (WaveletKind.HAAR, WaveletKind.DAUB4) and isinstance(pan, torch.Tensor) \
            and not _fusion._exact(None) and pan.is_cuda \
            and pan.dtype == torch.float32 and pan.dim() == 2 and bands \
            and all(isinstance(b, torch.Tensor) and b.dtype == torch.float32 for b in bands):
        h, w = pan.shape
        p_t = _plane(pan)
        m_t = [_plane(b) for b in bands]
        n = len(m_t)
        if h % 2 == 0 and w % 2 == 0 and \
                all(tuple(b.shape) == (h // 2, w // 2) for b in m_t) and \
                _scene_ok((*m_t, p_t), n, h, w, 2):
            if out is None:
                out = [torch.empty((h, w), dtype=torch.float32, device=p_t.device)
                       for _ in m_t]
            elif len(out) != n or any(o.shape != (h, w) or o.dtype != torch.float32 or
                                      o.device != p_t.device or not o.is_contiguous()
                                      for o in out):
                raise ValueError("out: one contiguous float32 (h, w) tensor per band on the "
                                 "PAN's device")
            code = 1 if method.kind == WaveletKind.HAAR else 2
            vec, flag = _fuse_quality_launch(p_t, m_t, out, code)
            return out, PendingReport((out, m_t, p_t), (None, vec, flag), n, 2)
    fused = _fusion.fuse(pan, ms, method)
    return fused, qnr_async(fused, ms, pan)


def fuse_and_qnr(pan, ms, method, *, one_pass: bool | None = None):
    """fuse(pan, ms, method) followed by qnr(fused, ms, pan); returns
    (fused, QualityReport).

    Haar scenes that qualify for the one-pass kernel (float32, 2..8
    half-size bands, H, W >= 64, W % 8 == 0) run SURVEY.md 8(f) row f1
    literally unless one_pass=False: the scoring kernel fuses each pixel
    itself and streams the fused bands out as it scores them, so they are
    never re-read (C ABI wf_fuse_quality_f32; bands bit-identical to
    fuse()'s, report identical to qnr()'s). Landsat, 6 bands: 3.05 ms one
    pass vs 3.17 ms for fuse() + qnr() (bench.py
    quality.fused_haar_fuse_and_report; round 1's one-pass kernel was the
    slower of the two at 3.6 ms until its row-pair loops stopped overflowing
    the instruction cache). D4 scenes that qualify take the same call, which
    runs the D4 fusion kernel and then the scoring kernel on its output (3.20
    ms, the fastest schedule measured: an SM-partitioned overlap of the two,
    WF_FQ_OVERLAP=1, measured 3.4 ms at best -- both kernels need every SM,
    profiles/r02_fq_overlap.log); one_pass=False forces fuse() + qnr()."""
    from . import fusion as _fusion
    from .wavelet import WaveletKind

    if not isinstance(method, _fusion.DwtReplace):
        raise TypeError(f"unknown fusion method {method!r}")
    is_t = isinstance(pan, torch.Tensor)
    p_shape = tuple(pan.shape) if is_t else np.shape(pan)
    bands = _bands(ms)
    fast = (one_pass is not False and method.kind in (WaveletKind.HAAR, WaveletKind.DAUB4)
            and not _fusion._exact(None)  # the exact default fuses in float64: fuse() then
            and len(p_shape) == 2
            and bands
            and all(_shape(b) == (p_shape[0] // 2, p_shape[1] // 2) for b in bands)
            and p_shape[0] % 2 == 0 and p_shape[1] % 2 == 0)
    if fast:
        # only a genuinely float32 PAN qualifies: a float64 / integer PAN fuses to
        # float64 (fusion.py:46-47), which this float32 kernel does not produce
        p_t = _device.to_device(pan, np.float32) if _device.is_f32(pan) else None
        m_t = [_plane(b) for b in bands] if p_t is not None else []
        n = len(m_t)
        h, w = p_shape
        if p_t is not None and p_t.dtype == torch.float32 and \
                _scene_ok((*m_t, p_t), n, h, w, 2) and all(t.dtype == torch.float32 for t in m_t):
            outs = [torch.empty((h, w), dtype=torch.float32, device=p_t.device) for _ in m_t]
            out, flag = _fuse_quality_launch(p_t, m_t, outs,
                                             1 if method.kind == WaveletKind.HAAR else 2)
            rep = (qnr(outs, m_t, p_t) if int(flag.item())
                   else _scene_report(out.cpu().numpy(), n, 2))
            return (outs if is_t else [_device.to_host(o) for o in outs]), rep
    if not is_t and not any(isinstance(b, torch.Tensor) for b in bands):
        # numpy in: the inputs go up once and the fused bands come down once
        # (fuse() on the host path, then qnr() of its numpy result, would move
        # the fused bands back up); same bits as the two separate calls
        out_dt = _device.np_out_dtype(pan)
        p_f = _device.to_device(pan, out_dt)
        m_f = [_device.to_device(b, out_dt) for b in bands]
        fused_t = _fusion.fuse(p_f, m_f, method)
        p_q = p_f if p_f.dtype == (torch.float32 if _device.is_f32(pan) else torch.float64) \
            else _plane(pan)
        m_q = [mf if mf.dtype == (torch.float32 if _device.is_f32(b) else torch.float64)
               else _plane(b) for mf, b in zip(m_f, bands)]
        rep = qnr(fused_t, m_q, p_q)
        return [_device.to_host(f) for f in fused_t], rep
    fused = _fusion.fuse(pan, ms, method)
    return fused, qnr(fused, ms, pan)
