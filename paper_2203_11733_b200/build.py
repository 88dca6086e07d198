"""In-tree build of the native libraries (sm_100a CUDA + C++ host).

    python -m paper_2203_11733_b200.build        # or __graft_entry__.build()

Outputs (git-ignored, shipped to the GPU box with the repo snapshot):
    paper_2203_11733_b200/lib/libgbem_gpu.so   CUDA kernels + the C-ABI of include/gbem_gpu.h
    paper_2203_11733_b200/lib/libgbem_host.so  C++ host (scene, partition, extraction driver, reports)
    paper_2203_11733_b200/lib/gbem             CLI
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = CSRC / "host"
LIB = PKG / "lib"
OBJ = LIB / "obj"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "nvcc")
CXX = os.environ.get("GBEM_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}"]
NVFLAGS += os.environ.get("GBEM_NVCC_EXTRA", "").split()  # experiments only (e.g. -DGBEM_FAR_MINB=5)
# Per-file extra flags: the assembly unit keeps the reference's operation order
# in the near-field closed forms (explicit fma() is still used in the far field).
EXTRA = {"gbem_assembly.cu": ["-fmad=false"]}
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", f"-I{INCLUDE}"]

CU_SOURCES = ["gbem_assembly.cu", "gbem_solver.cu", "gbem_block.cu", "gbem_selftest.cu", "gbem_pcg.cu", "gbem_capi.cu"]


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _headers(d: Path) -> list[Path]:
    return sorted(d.glob("*.cuh")) + sorted(d.glob("*.h")) + sorted(INCLUDE.glob("*.h"))


def build_gpu(force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdrs = _headers(CSRC)
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + NVFLAGS + EXTRA.get(src, []) + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(_run, jobs))
    so = LIB / "libgbem_gpu.so"
    if force or jobs or _stale(so, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", str(so)] + [str(o) for o in objs] + ["-lcudart", "-ldl"])
    return so


def build_host(force: bool = False) -> Path | None:
    srcs = sorted(HOST.glob("*.cpp"))
    if not srcs:
        return None
    OBJ.mkdir(parents=True, exist_ok=True)
    hdrs = sorted(HOST.glob("*.hpp")) + sorted(INCLUDE.glob("*.h"))
    jobs, objs = [], []
    lib_srcs = [s for s in srcs if s.name != "gbem_cli.cpp"]
    for s in srcs:
        o = OBJ / ("host_" + s.stem + ".o")
        if s.name != "gbem_cli.cpp":
            objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([CXX] + CXXFLAGS + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=max(1, min(8, len(jobs)))) as ex:
        list(ex.map(_run, jobs))
    so = LIB / "libgbem_host.so"
    gpu = LIB / "libgbem_gpu.so"
    if force or jobs or _stale(so, objs + [gpu]):
        _run([CXX, "-shared", "-o", str(so)] + [str(o) for o in objs]
             + [f"-L{LIB}", "-lgbem_gpu", f"-Wl,-rpath,$ORIGIN"])
    cli_src = HOST / "gbem_cli.cpp"
    if cli_src.exists():
        exe = LIB / "gbem"
        if force or _stale(exe, [cli_src, so]):
            _run([CXX] + CXXFLAGS + ["-o", str(exe), str(cli_src), f"-L{LIB}", "-lgbem_host",
                                     "-lgbem_gpu", "-Wl,-rpath,$ORIGIN"])
    del lib_srcs
    return so


def build(force: bool = False) -> None:
    build_gpu(force)
    build_host(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", LIB)
