"""Bind the B200 drop-in into an installed reference `wavefuse` package.

    import wavefuse
    from paper_1803_00737_b200 import integration
    handle = integration.install()      # every hot-path binding site -> sm_100a
    ...                                 # the reference's own code now runs on the GPU
    handle.uninstall()                  # restore the reference's functions

This is INTEGRATION.md section 1 as code: the binding sites SURVEY.md 8(b)
lists are rebound to paper_1803_00737_b200, with the reference's kinds,
exception classes and QualityReport translated at the boundary:

* wavefuse.fusion.fuse_dwt (fusion.py:128; `fuse` looks it up per band at
  fusion.py:182, so fuse / fuse_tiled / the CLI / the bench all route through
  it), the transforms (wavelet.py:131-164, bound into fusion.py:20),
  resample_bilinear (fusion.py:50, re-bound in metrics.py:15 and tiling.py)
  and the metrics (metrics.py:31-199);
* SURVEY.md 8(f) row f3, the cluster worker: WorkerServer.handle_task
  (cluster.py:297-299) is the reference's own hook; DWT tiles are fused on the
  GPU in the reference-exact mode (the wire result -- quantize() of the float
  planes, cluster.py:357-362 -- is then the reference worker's bytes), WA/IHS
  tiles stay on the CPU;
* row f4: fuse_tiled with per-tile wrap (tiling.py:213-273) and the PNM front
  end (imageio.py, and the names cli.py binds at import).

Nothing here computes: every rebinding calls the sm_100a library.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field

from . import errors as wf_errors

_ACTIVE: "Installed | None" = None
# DWT tiles fused on the GPU by any worker hook in this process
WORKER_TILES = {"count": 0}


@dataclass
class Installed:
    """What install() changed: (object, attribute, original value) triples and
    a count of calls routed to the GPU per name."""

    saved: list = field(default_factory=list)
    routed: dict = field(default_factory=dict)

    def set(self, obj, name: str, value) -> None:
        self.saved.append((obj, name, getattr(obj, name)))
        setattr(obj, name, value)

    def count(self, name: str) -> None:
        self.routed[name] = self.routed.get(name, 0) + 1

    def uninstall(self) -> None:
        global _ACTIVE
        for obj, name, value in reversed(self.saved):
            setattr(obj, name, value)
        self.saved.clear()
        if _ACTIVE is self:
            _ACTIVE = None


def gpu_handle_task(installed: Installed | None, cpu_handle):
    """WorkerServer.handle_task (cluster.py:297-299) on the B200: a DWT tile
    (8 bpp PAN + bands, tiling.py:163-172) is fused in the reference's own
    float64 sequence, so the float planes -- and the quantised wire bytes --
    equal the CPU worker's; other methods fall back to `cpu_handle`."""
    import wavefuse.fusion as F
    import wavefuse.wavelet as Wv

    from . import fusion as wf_fusion
    from .wavelet import WaveletKind

    kinds = {Wv.WaveletKind.HAAR: WaveletKind.HAAR, Wv.WaveletKind.DAUB4: WaveletKind.DAUB4}

    def handle_task(self, tile, method):
        if isinstance(method, F.DwtReplace):
            WORKER_TILES["count"] += 1
            if installed is not None:
                installed.count("worker_tiles")
            try:
                return wf_fusion.fuse_tile_quantized(tile.pan, tile.ms,
                                                     wf_fusion.DwtReplace(kinds[method.kind]),
                                                     exact=True)
            except wf_errors.FusionError as e:
                import wavefuse.errors as ref_errors

                raise getattr(ref_errors, type(e).__name__)(str(e)) from None
        return cpu_handle(self, tile, method)

    return handle_task


def install(keep_bench_pool: bool = True) -> Installed:
    """Rebind the reference's hot-path names to the B200 drop-in (idempotent:
    a second call returns the active handle). keep_bench_pool: the reference
    bench (and its acceptance criterion 8) measures the CPU thread-pool
    scaling of fuse_tiled, so wavefuse.bench keeps the reference's
    fuse_tiled (each tile still fuses on the GPU through fuse_dwt)."""
    global _ACTIVE
    if _ACTIVE is not None:
        return _ACTIVE
    import wavefuse
    import wavefuse.cli as Cli
    import wavefuse.cluster as Cl
    import wavefuse.errors as ref_errors
    import wavefuse.fusion as F
    import wavefuse.imageio as Io
    import wavefuse.metrics as M
    import wavefuse.tiling as T
    import wavefuse.wavelet as Wv

    import paper_1803_00737_b200 as wf

    inst = Installed()
    kinds = {Wv.WaveletKind.HAAR: wf.WaveletKind.HAAR, Wv.WaveletKind.DAUB4: wf.WaveletKind.DAUB4}

    def translate(fn, name):
        @functools.wraps(fn)
        def call(*args, **kwargs):
            inst.count(name)
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
    fwd2 = translate(wf.dwt2d_forward, "dwt2d_forward")
    inv2 = translate(wf.dwt2d_inverse, "dwt2d_inverse")
    fwd1 = translate(wf.dwt1d_forward, "dwt1d_forward")
    inv1 = translate(wf.dwt1d_inverse, "dwt1d_inverse")
    resample = translate(wf.resample_bilinear, "resample_bilinear")
    inst.set(F, "fuse_dwt", fuse_dwt)
    inst.set(F, "dwt2d_forward", fwd2)
    inst.set(F, "dwt2d_inverse", inv2)
    inst.set(F, "resample_bilinear", resample)
    inst.set(T, "resample_bilinear", resample)
    inst.set(Wv, "dwt1d_forward", fwd1)
    inst.set(Wv, "dwt1d_inverse", inv1)
    inst.set(Wv, "dwt2d_forward", fwd2)
    inst.set(Wv, "dwt2d_inverse", inv2)
    inst.set(M, "resample_bilinear", resample)
    for name in ("degrade", "q_index", "ergas", "d_lambda", "d_s", "qnr"):
        inst.set(M, name, translate(getattr(wf, name), name))

    # row f3: the B200-backed cluster worker
    inst.set(Cl.WorkerServer, "handle_task", gpu_handle_task(inst, Cl.WorkerServer.handle_task))

    # row f4: tiled fusion with per-tile wrap (plain and 8 bpp)
    cpu_tiled = T.fuse_tiled
    gpu_tiled = translate(wf.fuse_tiled, "fuse_tiled")

    def fuse_tiled(pan, ms, method, grid, workers=1, transfer_8bpp=False):
        if isinstance(method, F.DwtReplace):
            return gpu_tiled(pan, ms, wf.DwtReplace(kinds[method.kind]), grid, workers,
                             transfer_8bpp)
        return cpu_tiled(pan, ms, method, grid, workers, transfer_8bpp)

    inst.set(T, "fuse_tiled", fuse_tiled)
    inst.set(wavefuse, "fuse_tiled", fuse_tiled)
    if keep_bench_pool:
        import wavefuse.bench as Bn

        inst.set(Bn, "fuse_tiled", cpu_tiled)

    # row f4: the PNM front end and the CLI's data path (cli.py:113-165 binds
    # these names at import)
    for name in ("read_pnm", "write_pnm", "to_plane", "quantize"):
        fn = translate(getattr(wf, name), name)
        inst.set(Io, name, fn)
        inst.set(Cli, name, fn)
    inst.set(T, "pad_edge", translate(wf.pad_edge, "pad_edge"))
    inst.set(T, "pad_inputs", translate(wf.pad_inputs, "pad_inputs"))
    inst.set(Cli, "pad_inputs", T.pad_inputs)
    inst.set(Cli, "fuse_tiled", fuse_tiled)

    # the package's re-exports (wavefuse/__init__.py:18-51)
    for name in ("fuse_dwt", "resample_bilinear", "dwt1d_forward", "dwt1d_inverse",
                 "dwt2d_forward", "dwt2d_inverse", "degrade", "q_index", "ergas", "d_lambda",
                 "d_s", "qnr", "read_pnm", "write_pnm", "to_plane", "quantize", "pad_inputs"):
        if hasattr(wavefuse, name):
            inst.set(wavefuse, name, getattr(F, name, None) or getattr(Wv, name, None)
                     or getattr(Io, name, None) or getattr(T, name, None) or getattr(M, name))
    _ACTIVE = inst
    return inst


def gpu_worker(host: str = "127.0.0.1", port: int = 0):
    """A reference WorkerServer (cluster.py:286-394, wire protocol unchanged)
    whose DWT tiles fuse on the B200, without rebinding anything globally:
    `serve_forever()` it in a thread and point the reference master
    (run_master / MasterClient) at (worker.host, worker.port)."""
    import wavefuse.cluster as Cl

    worker = Cl.WorkerServer(host, port)
    worker.handle_task = gpu_handle_task(None, Cl.WorkerServer.handle_task).__get__(worker)
    return worker
