"""In-tree build of every native artefact.

  paper_2301_07457_b200/libtmg_gpu.so  -- the product: sm_100a CUDA + C ABI
  oracle/liboracle.so                  -- CPU checker (test infrastructure)
  oracle/_ref/libtopmg_ref.so          -- the unmodified reference, compiled
                                          from /root/reference when present

The .so files are git-ignored but travel to the GPU box with the gpurun
snapshot, so the box never rebuilds (and never needs /root/reference).
"""
from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["tmg_gpu.cu", "tmg_inputs.cpp"]
DEPS = SOURCES + ["tmg_device.cuh", "tmg_kernels.cuh", "tmg_march.cuh", "tmg_smarch.cuh", "tmg_smarch2.cuh", "tmg_stile.cuh", "tmg_oc.cuh", "tmg_poisson.cuh"]


def _stale(target: pathlib.Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps)


def build_gpu(force: bool = False, verbose: bool = False) -> pathlib.Path:
    out = PKG / "libtmg_gpu.so"
    deps = [CSRC / s for s in DEPS] + [ROOT / "include" / "tmg_gpu.h", pathlib.Path(__file__)]
    if not force and not _stale(out, deps):
        return out
    nvcc = NVCC if pathlib.Path(NVCC).exists() else shutil.which("nvcc")
    if not nvcc:
        raise RuntimeError("nvcc not found")
    cmd = [nvcc, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "static", "-o", str(out) + ".tmp", *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(str(out) + ".tmp", out)
    return out


def build_oracle(force: bool = False) -> None:
    odir = ROOT / "oracle"
    args = ["make", "-C", str(odir)]
    if force:
        args.append("-B")
    subprocess.run(args + ["liboracle.so"], check=True, stdout=subprocess.DEVNULL)
    ref = pathlib.Path(os.environ.get("TOPMG_REF_DIR", "/root/reference/proj"))
    if (ref / "src" / "solvers.cpp").exists():
        subprocess.run(args + ["ref", f"REF_DIR={ref}"], check=True, stdout=subprocess.DEVNULL)


def build_dropin(force: bool = False) -> None:
    """tests/cpp/dropin_check: the reference's own optimizer types and loop
    with the solve block served by include/topmg_gpu.hpp (test driver; needs
    the reference objects of oracle/_ref, so it is built where they exist)."""
    ref = pathlib.Path(os.environ.get("TOPMG_REF_DIR", "/root/reference/proj"))
    objs = [ROOT / "oracle" / "_ref" / f"{s}.o" for s in ("sparse", "grid", "density", "fem", "solvers", "mto")]
    if not (ref / "include").exists() or not all(o.exists() for o in objs):
        return
    src = ROOT / "tests" / "cpp" / "dropin_check.cpp"
    out = ROOT / "tests" / "cpp" / "dropin_check"
    lib = PKG / "libtmg_gpu.so"
    deps = [src, lib, ROOT / "include" / "topmg_gpu.hpp", *objs]
    if not force and not _stale(out, deps):
        return
    cmd = [shutil.which("g++") or "g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{ref / 'include'}",
           str(src), *map(str, objs), f"-L{PKG}", "-ltmg_gpu", "-Wl,-rpath,$ORIGIN/../../paper_2301_07457_b200",
           "-o", str(out)]
    subprocess.run(cmd, check=True)


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_oracle(force)
    build_dropin(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
