"""Build the sm_100a kernel library in-tree: paper_2509_19836_b200/_lib/libburst_b200.so.

Plain nvcc (no torch extension machinery): every ``csrc/*.cu`` is compiled for
``-gencode arch=compute_100a,code=sm_100a`` with ``-lineinfo`` and linked with a
static cudart, so the shared object has no link-time libcuda/libcudart
dependency and can be loaded (ctypes) on GPU-less hosts for symbol checks.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libburst_b200.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC,-O3",
    f"-I{INCLUDE}",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found: the burst-b200 kernels need CUDA 12.9 nvcc")
    return cand


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[Path]:
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(INCLUDE.glob("*.h"))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, defines: tuple[str, ...] = (),
          out: Path | None = None) -> Path:
    """Compile csrc/ into LIB.  ``defines`` (e.g. ``("BB_EXP_X",)``) and ``out`` build a
    developer variant library elsewhere (tools/variant.py); the product build takes neither."""
    lib = Path(out) if out else LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    out_dir = lib.parent
    out_dir.mkdir(parents=True, exist_ok=True)
    obj_dir = out_dir / ("obj" if out is None else lib.stem + "_obj")
    obj_dir.mkdir(exist_ok=True)
    exe = nvcc()
    extra = (["-Xptxas", "-v"] if ptxas_info else []) + [f"-D{d}" for d in defines]

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        cmd = [exe, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        if ptxas_info or verbose:
            sys.stderr.write(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [exe, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build(force=force, verbose="-v" in sys.argv, ptxas_info="--ptxas" in sys.argv))
