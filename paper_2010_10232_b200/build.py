"""Builds the in-tree sm_100a shared library ``libhelmdef_b200.so``.

nvcc cross-compiles for ``-gencode arch=compute_100a,code=sm_100a`` without a
GPU, so this runs in the CPU container as the driver's "does it build" check;
the resulting .so travels to the GPU box with the repo snapshot.
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
OUT = PKG / "libhelmdef_b200.so"
BUILD = PKG / "_build"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]

TOOL_SRC = ROOT / "tools" / "hd_cell.cpp"
TOOL = ROOT / "tools" / "hd_cell"
BENCH_SRC = ROOT / "tools" / "hd_bench.cpp"
BENCH = ROOT / "tools" / "hd_bench"


def nlohmann_include():
    """Directory holding nlohmann/json.hpp (the reference's JSON library; this
    image ships it inside site-packages, e.g. cudnn_frontend's thirdparty)."""
    env = os.environ.get("HD_NLOHMANN_INCLUDE")
    if env:
        return Path(env)
    import site
    roots = [Path(p) for p in site.getsitepackages()] + [Path("/usr/include"), Path("/usr/local/include")]
    for r in roots:
        for hit in sorted(r.glob("**/nlohmann/json.hpp")) if r.is_dir() else []:
            return hit.parent.parent
    return None
CU_SOURCES = ["solver.cu"]
CPP_SOURCES = ["host/banded.cpp", "host/assembly.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} exited {r.returncode}")
    return r


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.rglob("*.cuh")) + list(CSRC.rglob("*.hpp")) + list((ROOT / "include").glob("*.h"))
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = BUILD / (Path(src).stem + ".o")
        if _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, *COMMON, "-lineinfo", "-c", str(s), "-o", str(o)]
            if ptxas_info:
                cmd.insert(1, "-Xptxas=-v")
            r = _run(cmd)
            if verbose or ptxas_info:
                sys.stderr.write(r.stderr)
        objs.append(o)
    for src in CPP_SOURCES:
        s = CSRC / src
        o = BUILD / (Path(src).stem + ".cpp.o")
        if _stale(o, [s] + headers):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)])
        objs.append(o)
    if _stale(OUT, objs):
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(OUT),
              "-lcublas", "-lcusolver", "-lcudart", "-ldl"])
    # the C++ host mirror's cell tool (include/helmdef_b200.hpp), linked against
    # the in-tree library with a relative rpath so the built tree can move
    if TOOL_SRC.exists() and _stale(TOOL, [TOOL_SRC, OUT, ROOT / "include" / "helmdef_b200.hpp"]):
        _run(["g++", "-O2", "-std=c++17", "-Wall", "-I", str(ROOT / "include"), str(TOOL_SRC), "-o", str(TOOL),
              "-L", str(PKG), "-lhelmdef_b200", "-Wl,-rpath,$ORIGIN/../paper_2010_10232_b200"])
    # the helmbench CLI mirror (table / compare / solve) with the JSON harness
    inc = nlohmann_include()
    hdrs = [ROOT / "include" / "helmdef_b200.hpp", ROOT / "include" / "helmdef_b200_harness.hpp"]
    if inc is not None and BENCH_SRC.exists() and _stale(BENCH, [BENCH_SRC, OUT, *hdrs]):
        _run(["g++", "-O2", "-std=c++17", "-Wall", "-I", str(ROOT / "include"), "-I", str(inc), str(BENCH_SRC),
              "-o", str(BENCH), "-L", str(PKG), "-lhelmdef_b200", "-pthread",
              "-Wl,-rpath,$ORIGIN/../paper_2010_10232_b200"])
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, ptxas_info="-v" in sys.argv))
