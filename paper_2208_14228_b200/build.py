"""Build the sm_100a C-ABI library in-tree: paper_2208_14228_b200/libbittrain_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false:
-fmad=false because the reference (Python) never contracts a*b+c; the few
places where the reference's own libm fuses (glibc expm1 FMA variant) use
explicit __fma_rn in bt_libm.cuh.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libbittrain_b200.so"
BUILD = PKG / "_build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["bt_capi.cu", "bt_mlp.cu", "bt_reduce.cu", "bt_data.cu", "bt_gemm.cu", "bt_ffn.cu", "bt_bert.cu", "bt_cnn.cu", "bt_attn_tc.cu", "bt_embed.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "bittrain_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps if d.exists())


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    jobs = []
    for name in SOURCES:
        src, obj = CSRC / name, BUILD / (name + ".o")
        if force or _stale(obj, src):
            cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
            if verbose:
                sys.stderr.write(res.stderr)
    objs = [str(BUILD / (n + ".o")) for n in SOURCES]
    if force or not LIB.exists() or any(Path(o).stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", str(LIB), "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
