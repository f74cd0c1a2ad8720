"""Build the sm_100a C-ABI library `libconfkv_b200.so` in-tree with nvcc.

    python -m paper_2605_24786_b200.build [--force]

The shared library lands next to this file (git-ignored, but it travels to
the GPU box with the gpurun snapshot). Compiles only for sm_100a (B200).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libconfkv_b200.so"
SOURCES = ["abi.cu", "k1_confidence.cu", "k2_attention.cu", "k3_manage.cu", "decode_glue.cu"]
HEADERS = ["ckv_internal.cuh", "tc_i8.cuh"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "confkv_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)

    def compile_one(src):
        obj = build_dir / (src + ".o")
        # k3 (EMA, composite, quantizer) must not contract mul+add: the
        # reference rounds each product and sum separately.
        extra = ["-fmad=false"] if src in ("k3_manage.cu",) else []
        extra += os.environ.get("CKV_NVCC_EXTRA", "").split()
        cmd = [NVCC, ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj), *extra]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        return str(obj)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:   # one nvcc per translation unit
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([NVCC, ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
