"""Build libtdw.so in-tree for sm_100a (nvcc; no torch extension machinery)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libtdw.so"
SOURCES = ["coeff_table.cu", "assemble.cu", "march.cu", "fmm.cu", "capi.cu", "diag.cu", "tree.cu"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc, lib = Path(base) / "nccl" / "include", Path(base) / "nccl" / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return inc, lib
    raise RuntimeError("NCCL headers/library not found under site-packages/nvidia/nccl")


def nvcc():
    return shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


def build(verbose: bool = False, extra=()) -> Path:
    inc, lib = nccl_dirs()
    objs = []
    bdir = PKG / "build"
    bdir.mkdir(exist_ok=True)
    common = [nvcc(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "-lineinfo", "-Xcompiler", "-fPIC", f"-I{inc}", f"-I{ROOT / 'include'}", *extra]
    for src in SOURCES:
        obj = bdir / (src + ".o")
        objs.append(obj)
        deps = [CSRC / src] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "tdw.h"]
        stamp = bdir / (src + ".flags")  # rebuild when the extra flags change
        flags = " ".join(extra)
        same_flags = stamp.exists() and stamp.read_text() == flags
        if same_flags and obj.exists() and all(obj.stat().st_mtime >= p.stat().st_mtime for p in deps):
            continue
        stamp.write_text(flags)
        cmd = common + (["-Xptxas", "-v"] if verbose else []) + ["-c", str(CSRC / src), "-o", str(obj)]
        subprocess.run(cmd, check=True)
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(OUT),
           *map(str, objs), f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}", "-lcublas"]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(OUT)
