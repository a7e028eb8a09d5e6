"""In-tree build of the C-ABI library ``_lib/librinr_b200.so`` for sm_100a.

Plain nvcc, no torch headers: the library exports only the C functions in
``include/rinr_b200.h``.  Run ``python -m paper_2306_16699_b200.build`` (or
``__graft_entry__.build()``).  The built .so is git-ignored but travels to the
GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# RINR_LIB_DIR: build elsewhere (the -DRINR_CHECKED bounds-asserting build of
# tools/checked_build.sh goes to _lib_checked/)
LIB_DIR = Path(os.environ["RINR_LIB_DIR"]) if os.environ.get("RINR_LIB_DIR") else PKG / "_lib"
LIB = LIB_DIR / "librinr_b200.so"
SOURCES = [CSRC / "store.cpp", CSRC / "decode.cu", CSRC / "diag.cu", CSRC / "transforms.cu", CSRC / "fit.cu", CSRC / "fit_general.cu", CSRC / "writer.cu"]
HEADERS = [ROOT / "include" / "rinr_b200.h", ROOT / "include" / "rinr_b200_diag.h", ROOT / "include" / "rinr_b200_transforms.h", ROOT / "include" / "rinr_b200_encoder.h", ROOT / "include" / "rinr_b200_writer.h", CSRC / "rinr_internal.h", CSRC / "device_common.cuh", CSRC / "mma_chain.cuh", CSRC / "persist.cuh", CSRC / "tc_decode.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"] + os.environ.get("RINR_EXTRA_NVCC_FLAGS", "").split()


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    def compile_one(src: Path) -> str:
        obj = LIB_DIR / (src.stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cpp":
            cmd[1:1] = ["-x", "cu"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = LIB_DIR / (src.stem + ".ptxas.log")
        log.write_text(res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        if verbose:
            sys.stderr.write(res.stderr)
        return str(obj)

    # translation units compile independently: one nvcc per source, in parallel
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
