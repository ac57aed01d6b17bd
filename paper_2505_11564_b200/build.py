"""Builds libspecden_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2505_11564_b200.build [--force]

Every translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (no FMA contraction in
the parity-critical vector kernels is guaranteed by explicit __dadd_rn /
__dmul_rn intrinsics, not by a global flag).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libspecden_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-ffp-contract=off",
                "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
SOURCES = ["sd_vector.cu", "sd_host.cu", "sd_lanczos.cu", "sd_lanczos_tree.cu", "sd_gemm.cu", "sd_gemm_pair.cu", "sd_gpt_kernels.cu", "sd_mlp.cu",
           "sd_gpt.cu"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), ROOT / "include" / "specden_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = [CSRC / s for s in SOURCES if (CSRC / s).exists()]
    objs = [BUILD / (s.stem + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        if force or _stale(obj, src):
            cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-6000:]}")
            return True
        return False

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        changed = any(list(ex.map(compile_one, zip(srcs, objs))))
    if force or changed or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
