"""In-tree build of liblayerswap_b200.so (sm_100a) -- no JIT cache, no setuptools.

`build()` compiles every source under csrc/ and links one shared library at
paper_2605_11678_b200/_lib/liblayerswap_b200.so, which travels to the GPU box
with the repo snapshot.  Host policy code is compiled by g++ with
-ffp-contract=off (bit-exact CPython float semantics); CUDA sources by nvcc for
`-gencode arch=compute_100a,code=sm_100a` only.  Rebuilds are incremental by
mtime (sources + headers).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
OBJ_DIR = OUT_DIR / "obj"
LIB = OUT_DIR / "liblayerswap_b200.so"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-Wall", "-Wno-unused-function"]
NVCCFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                    "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA 12.9 toolkit is required to build liblayerswap_b200")


def _cuda_home() -> Path:
    return Path(_nvcc()).resolve().parent.parent


def _headers() -> list[Path]:
    return sorted(CSRC.rglob("*.h")) + sorted(CSRC.rglob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ... (exit {res.returncode})")


def build(verbose: bool = False) -> Path:
    """Compile csrc/*.cpp and csrc/*.cu into liblayerswap_b200.so."""
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    nvcc = _nvcc()
    cuda_inc = str(_cuda_home() / "include")
    objs: list[Path] = []
    jobs: list[tuple[str, list[str]]] = []
    for src in sorted(CSRC.glob("*.cpp")):
        obj = OBJ_DIR / (src.stem + ".cpp.o")
        if _stale(obj, [src] + headers):
            jobs.append((f"g++ {src.name}", ["g++", *CXXFLAGS, "-I", str(INCLUDE), "-I", cuda_inc,
                                              "-c", str(src), "-o", str(obj)]))
        objs.append(obj)
    for src in sorted(CSRC.glob("*.cu")):
        obj = OBJ_DIR / (src.stem + ".cu.o")
        if _stale(obj, [src] + headers):
            jobs.append((f"nvcc {src.name}", [nvcc, *NVCCFLAGS, "-I", str(INCLUDE), "-I", str(CSRC),
                                               "-c", str(src), "-o", str(obj)]))
        objs.append(obj)
    if jobs:
        from concurrent.futures import ThreadPoolExecutor
        if verbose:
            for name, _ in jobs:
                print("[build]", name)
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
            list(pool.map(lambda j: _run(j[1]), jobs))
    if _stale(LIB, objs):
        if verbose:
            print("[build] link", LIB.name)
        _run([nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
