"""Buffer plumbing between the reference-shaped API (numpy in, numpy out) and
the device library (torch CUDA tensors as allocations, torch streams).

The dtype rule is the reference's: output is float32 iff the input is float32,
otherwise float64 (wavelet.py:69-70, fusion.py:46-47); integer inputs promote
to float64 (test_wavelet.py:219-222).
"""

from __future__ import annotations

import atexit
import threading

import numpy as np
import torch

from . import _native

_tls = threading.local()
_ctxs: list[int] = []
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
    return torch.from_numpy(arr).to(dev)


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def host_ctx() -> int:
    """Per-thread wf_ctx for the host-buffer pipeline (re-entrant across
    threads: each thread owns its streams and staging slots)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        dev = require_cuda()
        ctx = _native.load().wf_ctx_create(dev.index, 0)
        if not ctx:
            _native.check(5)
        _tls.ctx = ctx
        with _ctx_lock:
            _ctxs.append(ctx)
    return ctx


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
