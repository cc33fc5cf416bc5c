"""In-tree build of libpdlp_b200.so (sm_100a) — invoked by __graft_entry__.build().

Each .cu compiles to an object in parallel, then one nvcc link produces
paper_2311_12180_b200/lib/libpdlp_b200.so with the CUDA runtime linked
statically, so the library only needs the driver at run time.

--fmad=false: the reference's x86-64 build never contracts a*b+c into an FMA,
and parity mode promises bitwise-equal iterates; the kernels are HBM-bound, so
the extra DMUL/DADD issue slots are free.
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
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libpdlp_b200.so"
OBJ_DIR = PKG / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    *ARCH,
    "-lineinfo",
    "--fmad=false",
    "-Xcompiler",
    "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas",
    "-O3",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-g"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _deps() -> list[Path]:
    return sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [
        PKG.parent / "include" / "pdlp_b200.h", Path(__file__)
    ]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
          defines: tuple[str, ...] = (), out: Path | None = None) -> Path:
    """Builds the library. `defines` / `out` make A/B variants of compile-time
    tuning constants (tools/build_variants.py); the product is LIB."""
    if not force and out is None and not defines and up_to_date():
        return LIB
    target = Path(out) if out is not None else LIB
    obj_dir = OBJ_DIR if out is None else OBJ_DIR / target.stem
    obj_dir.mkdir(parents=True, exist_ok=True)
    target.parent.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    extra = (["-Xptxas", "-v"] if ptxas_verbose else []) + [f"-D{d}" for d in defines]

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        if src.suffix == ".cpp":  # host-only C++ (LP I/O): the system g++
            cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
        else:
            cmd = [cc, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose or ptxas_verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = target.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-lz"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
    print(LIB)
