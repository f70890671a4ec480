"""In-tree build of the native libraries (no JIT cache: the .so files travel with the tree).

    libchgpu.so   nvcc, sm_100a only: kernels + context + C ABI (include/chgpu.h)
    libchsynth.so g++: synthetic dataset generator (tests / bench inputs)

`python -m paper_1805_08995_b200.build` builds both; `build_all()` is what
`__graft_entry__.build()` calls.  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
]

# translation units of libchgpu.so; the match kernel's variants are split so they compile in parallel
CHGPU_UNITS = ["chgpu.cu", "match_smem.cu", "match_global.cu", "match_guided.cu", "match_tiled.cu", "match_dbg.cu", "match_active.cu", "host_util.cpp",
               "residency.cpp"]
CHGPU_HEADERS = ["dev_types.cuh", "hash_kernels.cuh", "hash_tc.cuh", "join_kernels.cuh", "general_kernels.cuh", "match_kernels.cuh", "match_launch.cuh", "compact_kernels.cuh", "plan_tasks.hpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA extension is mandatory (no CPU fallback)")


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_chgpu(force: bool = False, verbose: bool = False) -> Path:
    from concurrent.futures import ThreadPoolExecutor

    target = PKG / "libchgpu.so"
    headers = [CSRC / h for h in CHGPU_HEADERS] + [ROOT / "include" / "chgpu.h"]
    objdir = CSRC / "_obj"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()

    def compile_unit(name: str) -> Path:
        src = CSRC / name
        obj = objdir / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            cmd = [nvcc, *NVCC_FLAGS, *os.environ.get("CHGPU_NVCC_EXTRA", "").split(), "-c", "-o", str(obj), str(src)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.run(cmd, check=True, cwd=str(CSRC))
        return obj

    with ThreadPoolExecutor(max_workers=len(CHGPU_UNITS)) as ex:
        objs = list(ex.map(compile_unit, CHGPU_UNITS))
    if force or _stale(target, objs):
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(target),
                        *map(str, objs)], check=True, cwd=str(CSRC))
    return target


def build_chsynth(force: bool = False) -> Path:
    target = PKG / "libchsynth.so"
    src = CSRC / "synth.cpp"
    if force or _stale(target, [src]):
        cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
        subprocess.run([cxx, "-std=gnu++17", "-O2", "-fPIC", "-shared", "-pthread", "-Wl,-Bsymbolic", "-Wl,--exclude-libs,ALL",
                        "-o", str(target), str(src)],
                       check=True)
    return target


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_chgpu(force, verbose)
    build_chsynth(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", PKG / "libchgpu.so", PKG / "libchsynth.so")
