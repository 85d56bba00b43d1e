"""pytest plugin: run the REFERENCE's own test suite against the B200 drop-in.

    PYTHONPATH=baseline/_ref:. python -m pytest baseline/_ref/tests \
        -p tools.conformance_plugin -q

Before test collection it rebinds the reference's hot-path names (the binding
sites listed in SURVEY.md 8(b)) to paper_1803_00737_b200, exactly as
INTEGRATION.md section 1 tells a maintainer to: wavefuse.fusion.fuse_dwt
(which routes fuse / fuse_tiled / the cluster worker / the CLI / the bench),
the transforms, resample_bilinear, and the metrics. Kinds, exception classes
and QualityReport are translated at the boundary. Nothing here computes: every
rebinding calls the sm_100a library.
"""

from __future__ import annotations

import functools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1803_00737_b200 as wf  # noqa: E402
from paper_1803_00737_b200 import errors as wf_errors  # noqa: E402

ROUTED: dict[str, int] = {}


def _install():
    import wavefuse
    import wavefuse.errors as ref_errors
    import wavefuse.fusion as F
    import wavefuse.metrics as M
    import wavefuse.tiling as T
    import wavefuse.wavelet as Wv

    kinds = {Wv.WaveletKind.HAAR: wf.WaveletKind.HAAR, Wv.WaveletKind.DAUB4: wf.WaveletKind.DAUB4}

    def translate(fn, name):
        @functools.wraps(fn)
        def call(*args, **kwargs):
            ROUTED[name] = ROUTED.get(name, 0) + 1
            args = [kinds.get(a, a) if isinstance(a, Wv.WaveletKind) else a for a in args]
            try:
                out = fn(*args, **kwargs)
            except wf_errors.FusionError as e:
                raise getattr(ref_errors, type(e).__name__)(str(e)) from None
            if isinstance(out, wf.QualityReport):
                out = M.QualityReport(ergas=out.ergas, q_per_band=out.q_per_band,
                                      d_lambda=out.d_lambda, d_s=out.d_s, qnr=out.qnr)
            return out
        return call

    fuse_dwt = translate(wf.fuse_dwt, "fuse_dwt")
    fwd2, inv2 = translate(wf.dwt2d_forward, "dwt2d_forward"), translate(wf.dwt2d_inverse, "dwt2d_inverse")
    fwd1, inv1 = translate(wf.dwt1d_forward, "dwt1d_forward"), translate(wf.dwt1d_inverse, "dwt1d_inverse")
    resample = translate(wf.resample_bilinear, "resample_bilinear")
    F.fuse_dwt = fuse_dwt
    F.dwt2d_forward, F.dwt2d_inverse = fwd2, inv2
    F.resample_bilinear = resample
    T.resample_bilinear = resample
    Wv.dwt1d_forward, Wv.dwt1d_inverse = fwd1, inv1
    Wv.dwt2d_forward, Wv.dwt2d_inverse = fwd2, inv2
    M.resample_bilinear = resample
    for name in ("degrade", "q_index", "ergas", "d_lambda", "d_s", "qnr"):
        setattr(M, name, translate(getattr(wf, name), name))
    # a B200-backed cluster worker. WorkerServer.handle_task
    # (cluster.py:297-299) is the reference's own hook; DWT tiles go to the GPU
    # (8 bpp tile -> float32 planes, tiling.py:163-172), WA/IHS stay on the CPU.
    import wavefuse.cluster as Cl

    cpu_handle = Cl.WorkerServer.handle_task

    def gpu_handle_task(self, tile, method):
        if isinstance(method, F.DwtReplace):
            ROUTED["worker_tiles"] = ROUTED.get("worker_tiles", 0) + 1
            return wf.fuse_tile_quantized(tile.pan, tile.ms, wf.DwtReplace(kinds[method.kind]))
        return cpu_handle(self, tile, method)

    Cl.WorkerServer.handle_task = gpu_handle_task

    # tiled fusion with per-tile wrap (plain and 8 bpp)
    cpu_tiled = T.fuse_tiled
    gpu_tiled = translate(wf.fuse_tiled, "fuse_tiled")

    def fuse_tiled(pan, ms, method, grid, workers=1, transfer_8bpp=False):
        if isinstance(method, F.DwtReplace):
            return gpu_tiled(pan, ms, wf.DwtReplace(kinds[method.kind]), grid, workers,
                             transfer_8bpp)
        return cpu_tiled(pan, ms, method, grid, workers, transfer_8bpp)

    T.fuse_tiled = fuse_tiled
    wavefuse.fuse_tiled = fuse_tiled
    # the reference bench (and its acceptance criterion 8) measures CPU-worker
    # scaling of its thread pool; keep that pool (each tile still fuses on the
    # GPU through the fuse_dwt rebinding above)
    import wavefuse.bench as Bn

    Bn.fuse_tiled = cpu_tiled

    # the PNM front end (imageio.py) and the CLI's data
    # path (cli.py:113-165 binds these names at import)
    import wavefuse.cli as Cli
    import wavefuse.imageio as Io

    for name in ("read_pnm", "write_pnm", "to_plane", "quantize"):
        setattr(Io, name, translate(getattr(wf, name), name))
        setattr(Cli, name, getattr(Io, name))
    T.pad_edge = translate(wf.pad_edge, "pad_edge")
    T.pad_inputs = translate(wf.pad_inputs, "pad_inputs")
    Cli.pad_inputs = T.pad_inputs
    Cli.fuse_tiled = fuse_tiled

    for name in ("fuse_dwt", "resample_bilinear", "dwt1d_forward", "dwt1d_inverse",
                 "dwt2d_forward", "dwt2d_inverse", "degrade", "q_index", "ergas", "d_lambda",
                 "d_s", "qnr", "read_pnm", "write_pnm", "to_plane", "quantize", "pad_inputs"):
        if hasattr(wavefuse, name):
            setattr(wavefuse, name, getattr(F, name, None) or getattr(Wv, name, None)
                    or getattr(Io, name, None) or getattr(T, name, None) or getattr(M, name))


def pytest_configure(config):
    _install()


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line("B200 drop-in calls routed: " +
                                ", ".join(f"{k}={v}" for k, v in sorted(ROUTED.items())))
