"""Build libvsb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python build.py            # incremental (per-file objects, rebuilt when sources change)
    python build.py --clean
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
PKG = ROOT / "paper_2605_15957_b200"
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libvsb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]


def _hdr_digest() -> str:
    h = hashlib.sha256()
    # every .cu too: vs_tc128.cu includes vs_tc.cu (one tile width per object)
    for p in sorted(list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(CSRC.glob("vs_tc.cu")) +
                    [ROOT / "include" / "vs_b200.h"]):
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _compile(src: Path, hdr: str) -> Path:
    digest = hashlib.sha256(src.read_bytes() + hdr.encode() + " ".join(FLAGS).encode()).hexdigest()[:16]
    obj = OBJ / f"{src.stem}.{digest}.o"
    if not obj.exists():
        for old in OBJ.glob(f"{src.stem}.*.o"):
            old.unlink()
        cmd = [NVCC, *ARCH, *FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = True) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr = _hdr_digest()
    srcs = sorted(CSRC.glob("*.cu"))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcuda"]
        subprocess.run(cmd, check=True)
        if verbose:
            print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    if "--clean" in sys.argv:
        import shutil
        shutil.rmtree(ROOT / "build", ignore_errors=True)
        LIB.unlink(missing_ok=True)
    build()
