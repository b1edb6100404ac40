"""Where does config 3's end-to-end time go? (diagnostic, not a bench line)

Times, on one GPU, with the bench's own workload object: the device step, the
end-to-end step (host queries + bitmap, host outputs), a bare pinned H2D copy
of the query batch, and the host wall time of each call.
Usage: python scripts/e2e_probe.py [config]
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402


def ev_time(fn, n):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / n
    return e0.elapsed_time(e1) / n, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, nargs="?", default=3)
    a = ap.parse_args()
    args = argparse.Namespace(gpus=1, steps=10, warmup=3, config=a.config, impl="ours", no_cpu=True,
                              cpu_budget=0, ref_budget=0, cand_slack=0, n_rows=0)
    cfg = dict(bench.CONFIGS[a.config])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    wl = (bench.IvfBf16Workload if cfg.get("bf16") else bench.IvfWorkload if "nlist" in cfg
          else bench.ExactWorkload)(args, cfg, 0, 1, dev)
    for _ in range(3):
        wl.step_device()
        wl.step_e2e()
    n = 10
    qd = torch.empty_like(wl.q_host, device=dev)
    print(f"device step      : {ev_time(wl.step_device, n)} (event ms, wall ms)")
    print(f"e2e step         : {ev_time(wl.step_e2e, n)}")
    print(f"H2D queries only : {ev_time(lambda: qd.copy_(wl.q_host, non_blocking=True), n)} "
          f"({wl.q_host.numel() * 4 / 1e6:.1f} MB)")
    if getattr(wl, "bits_host", None) is not None:
        bd = torch.empty_like(wl.bits_host, device=dev)
        print(f"H2D bitmap only  : {ev_time(lambda: bd.copy_(wl.bits_host, non_blocking=True), n)}")

    def upload_then_device():
        qd.copy_(wl.q_host, non_blocking=True)
        wl.step_device()
    print(f"H2D + device step: {ev_time(upload_then_device, n)}")


def interleaved_zero_copy(config=2, rounds=6):
    """e2e with zero-copy outputs on (any size) and off, interleaved in one
    process so clock drift hits both arms alike."""
    import os
    args = argparse.Namespace(gpus=1, steps=10, warmup=3, config=config, impl="ours", no_cpu=True,
                              cpu_budget=0, ref_budget=0, cand_slack=0, n_rows=0)
    cfg = dict(bench.CONFIGS[config])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    wl = (bench.IvfBf16Workload if cfg.get("bf16") else bench.IvfWorkload if "nlist" in cfg
          else bench.ExactWorkload)(args, cfg, 0, 1, dev)
    for _ in range(3):
        wl.step_device()
        wl.step_e2e()
    res = {"on": [], "off": [], "device": []}
    for _ in range(rounds):
        for arm, v in (("on", str(1 << 40)), ("off", "0")):
            os.environ["VS_ZERO_COPY_MAX"] = v
            wl.step_e2e()
            res[arm].append(ev_time(wl.step_e2e, 5)[0])
        res["device"].append(ev_time(wl.step_device, 5)[0])
    for arm, v in res.items():
        print(f"config {config} {arm:6s}: " + " ".join(f"{x:.3f}" for x in v) + f"  median {sorted(v)[len(v) // 2]:.3f} ms")


def interleaved_chunks(config=3, rounds=6, arms=("0", "2", "4")):
    """e2e with the IVF chunked query upload at 0 / 2 / 4 chunks, interleaved."""
    import os
    args = argparse.Namespace(gpus=1, steps=10, warmup=3, config=config, impl="ours", no_cpu=True,
                              cpu_budget=0, ref_budget=0, cand_slack=0, n_rows=0)
    cfg = dict(bench.CONFIGS[config])
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    wl = (bench.IvfBf16Workload if cfg.get("bf16") else bench.IvfWorkload)(args, cfg, 0, 1, dev)
    for _ in range(3):
        wl.step_device()
        wl.step_e2e()
    res = {a: [] for a in arms}
    res["device"] = []
    for _ in range(rounds):
        for a in arms:
            os.environ["VS_Q_CHUNKS"] = a
            wl.step_e2e()
            res[a].append(ev_time(wl.step_e2e, 5)[0])
        res["device"].append(ev_time(wl.step_device, 5)[0])
    for arm, v in res.items():
        print(f"config {config} chunks {arm:6s}: " + " ".join(f"{x:.3f}" for x in v)
              + f"  median {sorted(v)[len(v) // 2]:.3f} ms")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "chunks":
        interleaved_chunks(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    elif len(sys.argv) > 1 and sys.argv[1] == "zc":
        interleaved_zero_copy(int(sys.argv[2]) if len(sys.argv) > 2 else 2)
    else:
        main()
