"""Build the sm_100a shared library in-tree with nvcc (no torch extension
machinery: the library is a plain C-ABI `.so`, loaded with ctypes).

    python -m paper_1803_00737_b200._build          # build if stale
    python -m paper_1803_00737_b200._build --force  # rebuild
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libwavefuse_b200.so"
HEADER = ROOT / "include" / "wavefuse_b200.h"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-fmad=false",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
]
OBJ = PKG / "build"


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return path


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


# the checked variant (device-side ring/bounds invariants, wf_common.cuh
# WF_CHECK): a separate library and object directory, loaded only with
# WF_CHECKED=1
LIB_CHECKED = PKG / "libwavefuse_b200_checked.so"
OBJ_CHECKED = PKG / "build_checked"


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    built = lib.stat().st_mtime
    deps = sources() + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [HEADER]
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file),
    then link the shared library; the log of every step goes to build.log.
    checked=True builds the WF_CHECKS variant (LIB_CHECKED)."""
    lib = LIB_CHECKED if checked else LIB
    objdir = OBJ_CHECKED if checked else OBJ
    if not force and not stale(lib):
        return lib
    objdir.mkdir(exist_ok=True)
    inc = ["-I", str(ROOT / "include")]
    extra = ["-DWF_CHECKS"] if checked else []

    def compile_one(src: Path):
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *extra, *inc, "-c", "-o", str(obj), str(src)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, proc

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as pool:
        results = list(pool.map(compile_one, srcs))
    log_text = []
    failed = []
    for src, obj, cmd, proc in results:
        log_text.append(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        if proc.returncode != 0:
            failed.append((src, proc.stderr))
    tmp = lib.with_suffix(".so.tmp")
    if not failed:
        # peer.cu resolves cuMemGetAddressRange from libcuda at run time (-ldl)
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *[str(o) for _, o, _, _ in results], "-ldl"]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        log_text.append(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        if proc.returncode != 0:
            failed.append((lib, proc.stderr))
    log = PKG / ("build_checked.log" if checked else "build.log")
    log.write_text("\n".join(log_text))
    if failed:
        for _, err in failed:
            sys.stderr.write(err)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("\n".join(log_text))
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                checked="--checked" in sys.argv))
