"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Default workload = BASELINE.json configs[1] (config 2): exact filtered
top-100 over 10M x 1024 fp32 embeddings (41 GB resident in HBM), 10% Bernoulli
selectivity bitmap, 10k-query batch, squared L2, one B200. A step = one
search of the whole 10k-query batch. Under torchrun (N > 1) the 10M rows are
row-sharded across ranks (strong scaling), each rank searches its shard with
global row ids, and the per-rank [Q, k] results are all-gathered over NCCL and
merged by the library's merge kernel.

`value`  : queries/s with queries, bitmap and outputs resident in HBM.
`e2e`    : the same through the public API with pinned HOST buffers (query
           upload + bitmap upload + result download inside the timed region).
Other configs (--config 1/3) are available for measurement; the driver's
headline is config 2.

The CPU legs (`cpu_baseline`, `--impl reference`) time the oracle port of the
reference search (oracle/sqlvs_oracle.py: float64 pairwise + tie-rule top-k,
exactly the reference's arithmetic) on a bounded sample of the same workload
law and extrapolate linearly in rows (the reference's cost is O(Q*N*d)).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

CONFIGS = {
    1: dict(name="cfg1: Vec-H SF=0.1 filtered exact top-10, 100k x 384 fp32, TPC-H p_size<=5 bitmap, 1k queries",
            n=100_000, d=384, q=1000, k=10, sel=None),
    2: dict(name="cfg2: exact filtered top-100 over 10M x 1024 fp32, 10% Bernoulli bitmap, 10k-query batch",
            n=10_000_000, d=1024, q=10_000, k=100, sel=0.10),
    3: dict(name="cfg3: IVF-Flat nlist=16384 nprobe=32 top-10 over 10M x 1024 fp32, 1% bitmap, 10k queries",
            n=10_000_000, d=1024, q=10_000, k=10, sel=0.01, nlist=16384, nprobe=32),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- clocks sampling (nvidia-smi during the timed region) ---------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


# ---- workloads ---------------------------------------------------------------------------------

def pack_bits_torch(mask):
    import torch
    n = mask.numel()
    pad = (-n) % 32
    if pad:
        mask = torch.cat([mask, torch.zeros(pad, dtype=torch.bool, device=mask.device)])
    w = mask.view(-1, 32).to(torch.int64)
    shifts = torch.arange(32, device=mask.device, dtype=torch.int64)
    words = (w << shifts).sum(dim=1)
    return (words - ((words >> 31) << 32)).to(torch.int32).contiguous()  # two's complement uint32


def build_cfg2(rank, world, cfg):
    import torch

    from paper_2605_15957_b200 import synth
    from paper_2605_15957_b200.distributed import row_shard
    n, d, nq = cfg["n"], cfg["d"], cfg["q"]
    lo, hi = row_shard(n, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    # the same global collection on every world size: rows drawn in global
    # chunks, each rank keeps its slice
    t0 = time.time()
    data, centers = _device_slice(n, d, lo, hi, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(4242)
    mask = torch.rand(n, generator=g, device=dev) < cfg["sel"]
    mask_local = mask[lo:hi].contiguous()
    bits = pack_bits_torch(mask_local)
    queries = synth.device_queries(centers, nq, seed=7)
    torch.cuda.synchronize()
    log(f"[rank {rank}] generated {hi - lo} x {d} rows in {time.time() - t0:.1f}s; "
        f"selected {int(mask_local.sum())}")
    return dict(data=data, bits=bits, mask=mask_local, queries=queries, lo=lo, hi=hi,
                n_sel=int(mask_local.sum()), n_sel_total=int(mask.sum()))


def _device_slice(n, d, lo, hi, dev):
    import torch

    from paper_2605_15957_b200 import synth
    chunk = 1 << 20
    # regenerate global chunks covering [lo, hi) with per-chunk seeds
    g = torch.Generator(device=dev)
    g.manual_seed(42)
    c = torch.randn(64, d, generator=g, device=dev)
    c /= c.norm(dim=1, keepdim=True)
    out = torch.empty(hi - lo, d, device=dev)
    for ci in range(lo // chunk, (hi + chunk - 1) // chunk):
        a, b = ci * chunk, min(n, (ci + 1) * chunk)
        gg = torch.Generator(device=dev)
        gg.manual_seed(100_000 + ci)
        asg = torch.randint(0, 64, (b - a,), generator=gg, device=dev)
        v = c[asg] + 0.55 * torch.randn(b - a, d, generator=gg, device=dev)
        v /= v.norm(dim=1, keepdim=True)
        s, e = max(a, lo), min(b, hi)
        out[s - lo:e - lo] = v[s - a:e - a]
    del synth
    return out, c


# ---- CPU legs (oracle port; test infrastructure only) --------------------------------------------

_SAMPLE = {}


def _cpu_worker(qi):
    from oracle import sqlvs_oracle as O
    s = _SAMPLE
    # reference pipeline: the filtered side is gathered once (relops.py:112-113),
    # then enn_search scores it exhaustively in float64 (vecindex.py:109-132)
    O.enn_search(s["q"][qi:qi + 1], s["xs"], s["k"], row_ids=s["rows"])
    return qi


def cpu_sample(cfg, rows=262_144, seed=42):
    """Bounded sample of the config-2 law on the host: `rows` collection rows
    with the same selectivity, queries from the same mixture."""
    from paper_2605_15957_b200 import synth
    d = cfg["d"]
    x = synth.mixture_chunked(rows, d, seed=seed, chunk=1 << 16)
    rng = np.random.default_rng(seed)
    mask = rng.random(rows) < cfg["sel"]
    c = np.random.default_rng(np.random.SeedSequence([seed, 10])).standard_normal((64, d))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    qrng = np.random.default_rng(7)
    q = synth.mixture(qrng, c, qrng.integers(0, 64, 256), 0.165)
    return x, mask, q


def time_cpu_reference(cfg, budget_s=15.0, processes=1):
    """Reference search (oracle port) q/s on the sample, extrapolated to the
    full collection. processes > 1: query-sharded worker processes."""
    import multiprocessing as mp
    if "xs" not in _SAMPLE:
        x, mask, q = cpu_sample(cfg)
        rows_sel = np.flatnonzero(mask)
        _SAMPLE.update(xs=np.ascontiguousarray(x[rows_sel]), rows=rows_sel, q=q, k=cfg["k"],
                       n_rows=x.shape[0], n_sel=int(mask.sum()))
        del x
    q = _SAMPLE["q"]
    rows = _SAMPLE["n_rows"]
    done = 0
    t0 = time.perf_counter()
    if processes == 1:
        while True:
            _cpu_worker(done)
            done += 1
            if time.perf_counter() - t0 > budget_s or done >= len(q):
                break
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(processes) as pool:
            t0 = time.perf_counter()
            batch = processes
            while done < len(q):
                n = min(batch, len(q) - done)
                list(pool.imap_unordered(_cpu_worker, range(done, done + n)))
                done += n
                if time.perf_counter() - t0 > budget_s:
                    break
    el = time.perf_counter() - t0
    qps_sample = done / el
    qps_full = qps_sample * rows / cfg["n"]
    sample = (f"{done} queries x {rows} rows ({_SAMPLE['n_sel']} selected, d={cfg['d']}, k={cfg['k']}) "
              f"in {el:.1f}s; q/s extrapolated x{rows}/{cfg['n']} rows")
    return qps_full, sample, processes


# ---- our arm -----------------------------------------------------------------------------------

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2605_15957_b200 as vs
    from paper_2605_15957_b200 import _native as N
    from paper_2605_15957_b200.distributed import gpu_merge
    from paper_2605_15957_b200.vecindex import enn_search_raw

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W = build_cfg2(rank, world, cfg)
    k, nq, d = cfg["k"], cfg["q"], cfg["d"]
    col = vs.EmbeddingColumn.from_device(W["data"])
    ctx = N.Context.get(local)
    dev = torch.device("cuda", local)
    out_dev = (torch.empty((nq, k), dtype=torch.int64, device=dev),
               torch.empty((nq, k), dtype=torch.float64, device=dev),
               torch.empty((nq,), dtype=torch.int32, device=dev))
    q_host = W["queries"].cpu().pin_memory()
    bits_host = W["bits"].cpu().pin_memory()
    out_host = (torch.empty((nq, k), dtype=torch.int64).pin_memory(),
                torch.empty((nq, k), dtype=torch.float64).pin_memory(),
                torch.empty((nq,), dtype=torch.int32).pin_memory())
    merged_host = tuple(torch.empty_like(t).pin_memory() for t in out_host)

    def step_device():
        enn_search_raw(W["queries"], col, k, "squared_l2", row_filter=W["bits"], id_offset=W["lo"],
                       out=out_dev)
        if world > 1:
            from paper_2605_15957_b200.distributed import all_gather_topk
            gi, gd, gc = all_gather_topk(*out_dev)
            return gpu_merge(gi, gd, gc, k, "squared_l2")
        return out_dev

    def step_e2e():
        # public API with pinned host buffers: H2D of queries + bitmap and D2H of
        # the results happen inside the call
        if world == 1:
            enn_search_raw(q_host, col, k, "squared_l2", row_filter=bits_host, id_offset=W["lo"],
                           out=out_host)
            return
        enn_search_raw(q_host, col, k, "squared_l2", row_filter=bits_host, id_offset=W["lo"],
                       out=out_dev)
        from paper_2605_15957_b200.distributed import all_gather_topk
        gi, gd, gc = all_gather_topk(*out_dev)
        mi, md, mc = gpu_merge(gi, gd, gc, k, "squared_l2")
        merged_host[0].copy_(mi)
        merged_host[1].copy_(md)
        merged_host[2].copy_(mc)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    log(f"[rank {rank}] warmup {args.warmup}")
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    # correctness spot check on the first warm-up result (properties at full size)
    if args.warmup > 0:
        ids, dd, cc = out_dev
        assert int(cc.min()) == min(k, W["n_sel"]), "short result rows"
        assert bool((dd[:, 1:] >= dd[:, :-1]).all()), "distances not sorted"

    launches0 = ctx.stats()[N.STAT_LAUNCHES]
    ctx.set_option(N.OPT_TIMING, 1)
    ctx.kernel_times(reset=True)
    with ClockSampler(local) as clk:
        ms = timed(step_device, args.steps)
    kt = ctx.kernel_times(reset=True)
    ctx.set_option(N.OPT_TIMING, 0)
    launches = ctx.stats()[N.STAT_LAUNCHES] - launches0
    survivors = ctx.stats()[N.STAT_SURVIVORS]
    for _ in range(2):
        step_e2e()
    ctx.set_option(N.OPT_TIMING, 1)
    ctx.kernel_times(reset=True)
    t_host = time.perf_counter()
    ms_e2e = timed(step_e2e, args.steps)
    t_host = (time.perf_counter() - t_host) * 1e3
    kt_e2e = ctx.kernel_times(reset=True)
    ctx.set_option(N.OPT_TIMING, 0)

    ms_step = ms / args.steps
    qps = nq * args.steps / (ms / 1e3)
    qps_e2e = nq * args.steps / (ms_e2e / 1e3)
    # roofline of the dominant kernel (phase A scan): algorithmic FLOPs per
    # launch = 2 * Q * N_sel(local) * d
    scan_ns, scan_n = kt["enn_scan"]
    rr_ns, rr_n = kt["rerank"]
    sel_ns, sel_n = kt["select"]
    peaks = measured_peaks()
    flops = 2.0 * nq * W["n_sel"] * d
    achieved = flops / (scan_ns / max(scan_n, 1) / 1e9) / 1e12 if scan_n else None
    peak = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
    last_kernel = {1: "simt_fp32", 2: "tcgen05_bf16"}.get(ctx.stats()[N.STAT_LAST_ENN_KERNEL], "?")
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"cfg{args.config}:{last_kernel}")

    result = None
    if rank == 0:
        h2d = q_host.numel() * 4 + bits_host.numel() * 4
        d2h = sum(t.numel() * t.element_size() for t in out_host)
        result = {
            "metric": "filtered top-k queries/sec",
            "value": round(qps, 3),
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 3),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 storage; " + ("bf16 tcgen05 candidates" if last_kernel == "tcgen05_bf16"
                                        else "fp32 SIMT candidates") + "; f64 exact re-rank",
            "data": "synthetic (Vec-H mixture law generated on device; seeded Bernoulli bitmap)",
            "config": {"workload": cfg["name"], "n_rows": cfg["n"], "dim": d, "queries": nq, "k": k,
                       "selectivity": cfg["sel"], "n_selected": W["n_sel_total"],
                       "parallelism": f"row-shard x{world} + allgather/merge" if world > 1 else "single GPU",
                       "l2_flush": "inputs larger than L2 (41 GB collection vs 126 MB L2)",
                       "phase_a_kernel": last_kernel},
            "e2e": {"value": round(qps_e2e, 3), "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "kernel_ms_per_step": {c: round(v[0] / 1e6 / args.steps, 3) for c, v in kt.items() if v[1]},
            "e2e_kernel_ms_per_step": {c: round(v[0] / 1e6 / args.steps, 3) for c, v in kt_e2e.items() if v[1]},
            "e2e_host_ms_per_step": round(t_host / args.steps, 3),
            "survivors_per_query": round(survivors / nq, 2),
            "roofline": {"bound": "tensor", "kernel": f"enn_scan ({last_kernel})",
                         "achieved": round(achieved, 2) if achieved else None,
                         "peak": peak, "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4) if achieved else None,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (of measured)",
                         "algorithmic_flops_per_launch": flops,
                         "traffic": traffic},
            "clocks": clk.summary(),
        }
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu:
        qps_cpu, sample, cores = time_cpu_reference(cfg, budget_s=args.cpu_budget, processes=1)
        result["cpu_baseline"] = {"value": round(qps_cpu, 6), "unit": "queries/s", "cores": cores,
                                  "kind": "port", "sample": sample}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = min(os.cpu_count() or 1, 128)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    vals = []
    sample = ""
    for i in range(args.warmup + args.steps):
        qps, sample, _ = time_cpu_reference(cfg, budget_s=args.ref_budget, processes=procs)
        if i >= args.warmup:
            vals.append(qps)
    v = statistics.median(vals)
    print(json.dumps({
        "impl": "reference", "metric": "filtered top-k queries/sec", "value": round(v, 6),
        "unit": "queries/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (Vec-H mixture law, host sample)",
        "config": {"workload": cfg["name"]},
        "cpu_baseline": {"value": round(v, 6), "unit": "queries/s", "cores": procs, "kind": "port",
                         "sample": sample + f"; {procs} query-sharded processes"},
        "e2e": {"value": round(v, 6), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=8.0)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        if args.config != 2:
            raise SystemExit("only --config 2 is wired in bench.py so far")
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
