"""Buffer plumbing between the reference-shaped API (numpy in, numpy out) and
the device library (torch CUDA tensors as allocations, torch streams).

The dtype rule is the reference's: output is float32 iff the input is float32,
otherwise float64 (wavelet.py:69-70, fusion.py:46-47); integer inputs promote
to float64 (test_wavelet.py:219-222).
"""

from __future__ import annotations

import atexit
import contextlib
import threading

import numpy as np
import torch

from . import _native

_UPLOAD_MIN = 8 << 20  # bytes; smaller planes go through torch's copy
# PAN rows per host-pipeline strip (0 = the library default); WF_HOST_STRIP_ROWS
# overrides (each of the 3 slots pins (4 + 5 B) x rows x W bytes of staging)
_HOST_STRIP_ROWS = int(__import__("os").environ.get("WF_HOST_STRIP_ROWS", "0"))
_ctxs: list[int] = []
_free: dict[int, list[int]] = {}  # device index -> idle contexts bound to it
_ctx_lock = threading.Lock()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "wavefuse-b200 runs only on a CUDA device (sm_100a); there is no CPU fallback"
        )
    _native.load()
    return torch.device("cuda", torch.cuda.current_device())


def is_f32(x) -> bool:
    if isinstance(x, torch.Tensor):
        return x.dtype == torch.float32
    return np.asarray(x).dtype == np.float32


def np_out_dtype(x):
    return np.float32 if is_f32(x) else np.float64


def torch_dtype(np_dtype) -> torch.dtype:
    return torch.float32 if np_dtype == np.float32 else torch.float64


def as_host(x) -> np.ndarray:
    return x if isinstance(x, np.ndarray) else np.asarray(x)


def to_device(x, np_dtype) -> torch.Tensor:
    """Contiguous CUDA tensor of dtype np_dtype holding x (no copy when x is
    already such a tensor)."""
    dev = require_cuda()
    tdt = torch_dtype(np_dtype)
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(dev)
        return t.to(tdt).contiguous()
    arr = np.ascontiguousarray(np.asarray(x), dtype=np_dtype)
    if arr.nbytes < _UPLOAD_MIN:
        return torch.from_numpy(arr).to(dev)
    # large planes: the library's staged, multi-threaded upload (wf_ctx_upload)
    t = torch.empty(arr.shape, dtype=tdt, device=dev)
    with host_ctx() as ctx:
        _native.check(_native.load().wf_ctx_upload(ctx, t.data_ptr(), arr.ctypes.data, arr.nbytes,
                                                   stream_ptr()))
    return t


def to_host(t: torch.Tensor) -> np.ndarray:
    """A CUDA tensor as a fresh numpy array (`.cpu().numpy()`); planes of 8 MB
    and more come down through the library's staged, multi-threaded
    download (wf_ctx_download)."""
    if not t.is_cuda or t.numel() * t.element_size() < _UPLOAD_MIN:
        return t.cpu().numpy()
    t = t.contiguous()
    out = np.empty(tuple(t.shape), dtype=np.dtype(str(t.dtype).replace("torch.", "")))
    with host_ctx() as ctx:
        _native.check(_native.load().wf_ctx_download(ctx, out.ctypes.data, t.data_ptr(),
                                                     out.nbytes, stream_ptr()))
    return out


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


@contextlib.contextmanager
def host_ctx():
    """Borrow a wf_ctx (streams + device slots + pinned staging) for one
    host-buffer call. Contexts are pooled, not thread-local: concurrent
    callers get distinct contexts (the library is re-entrant per context) and
    later callers -- e.g. the fresh ThreadPoolExecutor threads of the
    reference's fuse_tiled (tiling.py:185-189) -- reuse warm ones instead of
    re-allocating pinned memory."""
    dev = require_cuda()  # the caller's current device: contexts are per device
    with _ctx_lock:
        pool = _free.setdefault(dev.index, [])
        ctx = pool.pop() if pool else None
    if ctx is None:
        ctx = _native.load().wf_ctx_create(dev.index, _HOST_STRIP_ROWS)
        if not ctx:
            _native.check(5)
        with _ctx_lock:
            _ctxs.append(ctx)
    try:
        yield ctx
    finally:
        with _ctx_lock:
            _free[dev.index].append(ctx)


@atexit.register
def _release() -> None:
    lib = _native._lib
    if lib is None:
        return
    with _ctx_lock:
        for c in _ctxs:
            try:
                lib.wf_ctx_destroy(c)
            except Exception:
                pass
        _ctxs.clear()
        _free.clear()
