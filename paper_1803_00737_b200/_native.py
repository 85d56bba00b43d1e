"""ctypes binding of the sm_100a C-ABI library (include/wavefuse_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises. Device buffers and streams come
from PyTorch (plumbing only); all compute happens in libwavefuse_b200.so.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading
from pathlib import Path

from . import errors

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libwavefuse_b200.so"
if os.environ.get("WF_CHECKED", "") not in ("", "0"):
    # the device-side-invariant build (_build.py --checked), for test runs
    LIB_PATH = _PKG / "libwavefuse_b200_checked.so"
HEADER_PATH = _PKG.parent / "include" / "wavefuse_b200.h"

HAAR, DAUB4 = 1, 2

_ERR = {
    1: ValueError,
    2: errors.OddDimension,
    3: errors.TooSmall,
    4: errors.DimensionMismatch,
    5: errors.CudaError,
    6: errors.BandCountMismatch,
    7: errors.OddLength,
    8: errors.TooShort,
    9: errors.NotDivisible,
    10: errors.ChannelOutOfRange,
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

c_int, c_i64, c_u32, c_u64 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
c_vp = ctypes.c_void_p
c_vpp = ctypes.POINTER(ctypes.c_void_p)


def header_symbols() -> list[str]:
    """Every function the public header declares (used by the export test)."""
    text = HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wf_[a-z0-9_]+)\s*\(", text)))


def _declare(lib: ctypes.CDLL) -> None:
    sig = {}
    for t in ("f32", "f64"):
        sig[f"wf_fuse_dwt_{t}"] = [c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_int, c_int, c_vp]
        sig[f"wf_fuse_bands_{t}"] = [c_int, c_vp, c_i64, c_vpp, c_i64, c_vpp, c_i64, c_int, c_int,
                                     c_int, c_vp]
        sig[f"wf_fuse_strip_{t}"] = [c_int, c_vp, c_i64, c_vp, c_vp, c_i64, c_vpp, c_vpp, c_i64,
                                     c_vpp, c_i64, c_int, c_int, c_int, c_vp]
        sig[f"wf_fuse_host_{t}"] = [c_vp, c_int, c_vp, c_vpp, c_vpp, c_int, c_int, c_int]
        sig[f"wf_fuse_strip_exact_{t}"] = sig[f"wf_fuse_strip_{t}"]
        for d in ("forward", "inverse"):
            sig[f"wf_dwt2d_{d}_{t}"] = [c_int, c_vp, c_i64, c_vp, c_i64, c_int, c_int, c_vp]
            sig[f"wf_dwt_rows_{d}_{t}"] = [c_int, c_vp, c_i64, c_vp, c_i64, c_int, c_int, c_vp]
        sig[f"wf_resample_bilinear_{t}"] = [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_int, c_int,
                                            c_vp]
    sig["wf_synth_plane_f32"] = [c_vp, c_i64, c_int, c_int, c_u64, c_u32, c_int, c_int, c_vp]
    sig["wf_fuse_bands_u8"] = sig["wf_fuse_bands_f32"]
    sig["wf_fuse_strip_u8"] = sig["wf_fuse_strip_f32"]
    sig["wf_fuse_host_u8"] = sig["wf_fuse_host_f32"]
    sig["wf_u8_to_f32"] = [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_vp]
    sig["wf_quantize_f32"] = [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_vp]
    sig["wf_quantize_f64"] = sig["wf_quantize_f32"]
    sig["wf_fuse_dwt_exact_f32"] = [c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_int, c_int,
                                    c_vp, c_vp]
    sig["wf_fuse_dwt_exact_f64"] = sig["wf_fuse_dwt_exact_f32"]
    sig["wf_fuse_bands_exact_f32"] = [c_int, c_vp, c_i64, c_vpp, c_i64, c_vpp, c_i64, c_int, c_int,
                                      c_int, c_vp, c_vp]
    sig["wf_fuse_bands_exact_f64"] = sig["wf_fuse_bands_exact_f32"]
    for t in ("f32", "f64"):
        sig[f"wf_raster_to_plane_{t}"] = [c_vp, c_int, c_int, c_int, c_int, c_vp, c_i64, c_int,
                                          c_int, c_vp]
        sig[f"wf_pad_edge_{t}"] = [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_int, c_int, c_vp]
        sig[f"wf_planes_to_raster_{t}"] = [c_vpp, c_int, c_i64, c_int, c_int, c_vp, c_vp]
    sig["wf_ipc_export"] = [c_vp, c_vp, ctypes.POINTER(c_u64)]
    sig["wf_ipc_open"] = [c_vp, ctypes.POINTER(c_vp)]
    sig["wf_ipc_close"] = [c_vp]
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int
    lib.wf_version.restype = ctypes.c_char_p
    lib.wf_last_error.restype = ctypes.c_char_p
    lib.wf_launch_count.restype = c_i64
    lib.wf_tuning_reload.restype = c_int
    lib.wf_checked_build.restype = c_int
    lib.wf_check_selftest.restype = c_int
    lib.wf_ctx_create.argtypes = [c_int, c_int]
    lib.wf_ctx_create.restype = c_vp
    lib.wf_ctx_upload.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp]
    lib.wf_ctx_upload.restype = c_int
    lib.wf_ctx_download.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp]
    lib.wf_ctx_download.restype = c_int
    lib.wf_ctx_set_exact.argtypes = [c_vp, c_int]
    lib.wf_ctx_set_exact.restype = c_int
    lib.wf_ctx_destroy.argtypes = [c_vp]
    lib.wf_ctx_destroy.restype = None
    _declare_quality(lib)


def _declare_quality(lib: ctypes.CDLL) -> None:
    sig = {
        "wf_resample_bilinear_f32_to_f64": ([c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_int, c_int,
                                             c_vp], c_int),
        "wf_q_index_workspace_bytes": ([c_int, c_int], c_i64),
        "wf_q_index": ([c_vp, c_int, c_i64, c_vp, c_int, c_i64, c_int, c_int, c_vp, c_vp, c_int,
                        c_vp], c_int),
        "wf_degrade": ([c_vp, c_int, c_i64, c_int, c_int, c_int, c_vp, c_i64, c_vp], c_int),
        "wf_ergas_workspace_bytes": ([c_int, c_int], c_i64),
        "wf_quality_scene_workspace_bytes": ([c_int, c_int, c_int], c_i64),
        "wf_quality_scene_f32": ([c_vpp, c_vpp, c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_int,
                                  c_vp, c_vp, c_vp, c_vp], c_int),
        "wf_quality_scene_f64": ([c_vpp, c_vpp, c_vp, c_i64, c_i64, c_i64, c_int, c_int, c_int,
                                  c_vp, c_vp, c_vp, c_vp], c_int),
        "wf_ergas_band": ([c_vp, c_int, c_i64, c_vp, c_int, c_i64, c_int, c_int, c_int, c_vp,
                           c_vp, c_vp], c_int),
        "wf_fuse_quality_f32": ([c_int, c_vp, c_i64, c_vpp, c_i64, c_vpp, c_i64, c_int, c_int,
                                 c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load() -> ctypes.CDLL:
    """Load (once) the in-tree library. Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH.name} is not built; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            _declare(lib)
            _lib = lib
        return _lib


def check(rc: int) -> None:
    if rc:
        msg = load().wf_last_error().decode(errors="replace")
        raise _ERR.get(rc, RuntimeError)(msg)


def reload_tuning() -> None:
    """Re-read the WF_* tuning environment (the library reads it once)."""
    if _lib is not None:
        _lib.wf_tuning_reload()


def launch_count() -> int:
    return int(load().wf_launch_count())


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
