"""Build recipe for the sm_100a C-ABI library ``libnar_b200.so``.

Every CUDA source under ``csrc/`` is compiled by nvcc for
``-gencode arch=compute_100a,code=sm_100a`` (never the generic compute_100
PTX pass, which rejects tcgen05) and linked into one shared library in the
package directory, so the built file travels with the repository snapshot.

raster.cu is compiled with ``-fmad=false``: the render arithmetic must keep
the reference's no-contraction float semantics (pkg/setup.py:23-25).
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
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "nar_b200"
LIB = PKG / "libnar_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          f"-I{INCLUDE}", f"-I{CSRC}", "--expt-relaxed-constexpr"]
PER_FILE = {"raster.cu": ["-fmad=false"], "gsplat.cu": ["-fmad=false"]}


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libnar_b200.so")
    return cand


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps_mtime() -> float:
    files = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _compile(src: Path, verbose: bool) -> Path:
    obj = BUILD / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= _deps_mtime():
        return obj
    # NAR_NVCC_EXTRA: extra flags for experiment builds (e.g. -DNAR_TC_TRACE); such a
    # build goes to another directory via NAR_BUILD_DIR so the product objects stay
    extra = os.environ.get("NAR_NVCC_EXTRA", "").split()
    cmd = [_nvcc(), *ARCH, *COMMON, *PER_FILE.get(src.name, []), *extra, "-c", str(src), "-o",
           str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu and link libnar_b200.so; returns the library path."""
    BUILD.mkdir(parents=True, exist_ok=True)
    if force:
        for o in BUILD.glob("*.o"):
            o.unlink()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if LIB.exists() and not force and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


C_CONSUMER_SRC = ROOT / "tests" / "c" / "abi_consumer.c"
C_CONSUMER = ROOT / "tests" / "c" / "abi_consumer"


def build_c_consumer() -> Path | None:
    """gcc the plain-C ABI consumer (tests/c/abi_consumer.c) against the header
    and libnar_b200.so -- proof that the boundary needs no Python or C++."""
    if not C_CONSUMER_SRC.exists():
        return None
    cuda = Path(_nvcc()).resolve().parent.parent
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", f"-I{INCLUDE}", f"-I{cuda / 'include'}",
           str(C_CONSUMER_SRC), "-o", str(C_CONSUMER), f"-L{PKG}", "-lnar_b200",
           f"-L{cuda / 'lib64'}", "-lcudart", "-Wl,-rpath,$ORIGIN/../../paper_2407_19097_b200",
           f"-Wl,-rpath,{cuda / 'lib64'}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"C consumer build failed:\n{res.stderr}")
    return C_CONSUMER


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
