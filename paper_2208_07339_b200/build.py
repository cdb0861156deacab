"""Build the in-tree sm_100a shared library ``_lib/libllmint8_sm100.so``.

nvcc cross-compiles for ``-gencode arch=compute_100a,code=sm_100a`` (no GPU
needed). The library exports the C ABI of ``include/llmint8.h`` and links
cudart statically, so it only needs the NVIDIA driver at run time.

    python -m paper_2208_07339_b200.build [--force] [--verbose] [--devtools]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB_NAME = "libllmint8_sm100.so"
SOURCES = ["capi.cu", "prologue.cu", "weights.cu", "gemm_sm100.cu", "decode_sm100.cu", "siblings.cu",
           "peak_sm100.cu", "f32path.cu", "swapab_sm100.cu"]
HEADERS = ["kernels.cuh", "sm100_ptx.cuh", "quant_common.cuh", "percall_dev.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found (need CUDA 12.9 for sm_100a)")


def lib_path(devtools: bool = False) -> Path:
    """The production library, or the dev build (timeline stamps, wait counters)."""
    return (OUT_DIR / "dev" if devtools else OUT_DIR) / LIB_NAME


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, devtools: bool = False) -> Path:
    out = lib_path(devtools).parent
    out.mkdir(parents=True, exist_ok=True)
    objdir = out / "obj"
    objdir.mkdir(exist_ok=True)
    headers = [CSRC / h for h in HEADERS] + [ROOT / "include" / "llmint8.h"]
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
    if verbose:
        flags += ["-Xptxas", "-v"]
    if devtools:  # scripts/*_timeline.py, I8MM_DBG_EPI: never the shipped library
        flags += ["-DI8MM_GEMM_DEVTOOLS"]
    cc = nvcc()

    def compile_one(src: str) -> Path:
        s = CSRC / src
        o = objdir / (s.stem + ".o")
        if force or _stale(o, [s] + headers):
            cmd = [cc, *flags, "-c", str(s), "-o", str(o)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
            if verbose and (r.stdout or r.stderr):
                print(r.stdout, r.stderr, file=sys.stderr)
        return o

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    lib = lib_path(devtools)
    if force or _stale(lib, objs):
        cmd = [cc, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--devtools", action="store_true", help="dev build into _lib/dev/")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, devtools=a.devtools))
