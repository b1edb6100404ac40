"""Run a few searches of one bench config with the profiling library and print
the re-rank kernel's average cycles per CTA by phase."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_15957_b200 import _native as N  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
args = type("A", (), {"config": cfg, "cpu_budget": 1.0})()
torch.cuda.set_device(0)
conf = dict(bench.CONFIGS[cfg])
if len(sys.argv) > 3:   # e.g. "2 1000000 1.0": same selected-row count from a 4 GB collection
    conf.update(n=int(sys.argv[2]), sel=float(sys.argv[3]))
wl = (bench.IvfWorkload if "nlist" in conf else bench.ExactWorkload)(
    args, conf, 0, 1, torch.device("cuda", 0))
lib = N.load()
lib.vs_debug_rerank_profile.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(8, np.uint64)
for _ in range(2):
    wl.step_device()
torch.cuda.synchronize()
lib.vs_debug_rerank_profile(buf.ctypes.data, 1)
steps = 3
for _ in range(steps):
    wl.step_device()
torch.cuda.synchronize()
lib.vs_debug_rerank_profile(buf.ctypes.data, 1)
names = ["setup", "gather", "select", "score", "topk"]
ctas = wl.nq * steps * (2 if "nlist" in conf else 1)
for i, n in enumerate(names):
    print(f"{n:8s} {buf[i] / ctas:12.0f} cycles/CTA")
print(f"candidates {buf[5] / ctas:10.0f} per CTA, live (key <= pre) {buf[6] / ctas:10.0f}")
