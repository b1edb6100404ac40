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
            id=1, n=100_000, d=384, q=1000, k=10, sel=None),
    2: dict(name="cfg2: exact filtered top-100 over 10M x 1024 fp32, 10% Bernoulli bitmap, 10k-query batch",
            id=2, n=10_000_000, d=1024, q=10_000, k=100, sel=0.10),
    3: dict(name="cfg3: IVF-Flat nlist=16384 nprobe=32 top-10 over 10M x 1024 fp32, 1% bitmap, 10k queries",
            id=3, n=10_000_000, d=1024, q=10_000, k=10, sel=0.01, nlist=16384, nprobe=32),
    4: dict(name="cfg4: IVF-Flat bf16 50M x 768, nlist=16384 nprobe=64 top-10, unfiltered, 10k queries, "
                 "sharded by list", id=4, n=50_000_000, d=768, q=10_000, k=10, sel=None, nlist=16384,
            nprobe=64, bf16=True, cpu_queries=4),
    5: dict(name="cfg5 B: exact filtered top-100 over 100M x 768 f32 row-sharded over 8 GPUs; each GPU's "
                 "12.5M-row shard (38.4 GB) resident in pinned HOST memory and streamed per search",
            id=5, n=100_000_000, d=768, q=10_000, k=100, sel=0.10, shards=8, host=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- clocks sampling (nvidia-smi during the timed region) ---------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled from a thread every ~2 ms (so even a 10 ms region gets samples;
    ctypes releases the GIL during library calls), else `nvidia-smi -lms 50`."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, reasons) from NVML
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.handle = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM))
            self._sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
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

    def _sample(self):
        nv = self.nvml
        sm = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((sm, {n for n, b in zip(self.NAMES, bits) if r & b}))

    def _poll(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            self._sample()
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if self.nvml is not None:
            sm = [x[0] for x in self.samples]
            reasons = set().union(*[x[1] for x in self.samples]) if self.samples else set()
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


# ---- workloads ---------------------------------------------------------------------------------

def pack_bits_torch(mask):
    from paper_2605_15957_b200.synth import pack_bits_torch as _p
    return _p(mask)


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
    from paper_2605_15957_b200.synth import device_rows
    return device_rows(n, d, lo, hi, dev)


def _device_slice_bf16(n, d, lo, hi, dev):
    """Rows [lo, hi) drawn chunk by chunk straight into bfloat16 (the float32
    collection would not fit next to the index)."""
    import torch

    from paper_2605_15957_b200.synth import device_rows
    return device_rows(n, d, lo, hi, dev, dtype=torch.bfloat16)


# ---- CPU legs (oracle port; test infrastructure only) --------------------------------------------

_SAMPLE = {}


def _ref_sqlvs():
    """The unmodified reference package shipped as oracle/_ref/sqlvs (copied by
    oracle/build_ref.py in the build container), or None."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "sqlvs" / "vecindex.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import sqlvs.table
    import sqlvs.vecindex
    return sqlvs


def _cpu_worker(qi):
    s = _SAMPLE
    # reference pipeline: the filtered side is gathered once (relops.py:112-113),
    # then enn_search scores it exhaustively in float64 (vecindex.py:109-132):
    # the reference's own code when shipped (oracle/_ref), else the oracle port
    ref = s.get("ref")
    if ref is not None:
        ref.vecindex.enn_search(ref.table.EmbeddingColumn(s["q"][qi:qi + 1]), s["ref_col"],
                                ref.vecindex.SearchParams(k=s["k"]))
        return qi
    from oracle import sqlvs_oracle as O
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


def time_cpu_reference(cfg, budget_s=15.0, processes=1, use_reference=False):
    """Reference search (oracle port) q/s on the sample, extrapolated to the
    full collection. processes > 1: query-sharded worker processes."""
    import multiprocessing as mp
    if "xs" not in _SAMPLE:
        x, mask, q = cpu_sample(cfg)
        rows_sel = np.flatnonzero(mask)
        _SAMPLE.update(xs=np.ascontiguousarray(x[rows_sel]), rows=rows_sel, q=q, k=cfg["k"],
                       n_rows=x.shape[0], n_sel=int(mask.sum()))
        del x
        ref = _ref_sqlvs() if use_reference else None
        if ref is not None:
            _SAMPLE.update(ref=ref, ref_col=ref.table.EmbeddingColumn(_SAMPLE["xs"]))
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

class Harness:
    """Barrier + CUDA-event timing on the launching stream, max over ranks."""

    def __init__(self, world, dev):
        self.world, self.dev = world, dev

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(self, fn, steps):
        import torch
        import torch.distributed as dist
        self.barrier()
        stream = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        self.barrier()
        ms = e0.elapsed_time(e1)
        if self.world > 1:
            t = torch.tensor([ms], device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms


def _pinned_like(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype).pin_memory()


class ExactWorkload:
    """Configs 1 and 2: filtered exact top-k (enn_search with a row bitmap).
    cfg2 row-shards the collection across ranks (strong scaling, NCCL
    all-gather + merge kernel); cfg1 is small, so ranks are replicas."""

    def __init__(self, args, cfg, rank, world, dev):
        import torch

        import paper_2605_15957_b200 as vs
        self.cfg, self.rank, self.world, self.dev = cfg, rank, world, dev
        self.k, self.nq, self.d = cfg["k"], cfg["q"], cfg["d"]
        self.replicas = args.config == 1
        if args.config == 1:
            from paper_2605_15957_b200 import synth
            emb, mask, q = synth.config1(cfg["n"])
            self.host_sample = (emb, mask, q)
            data = torch.from_numpy(np.ascontiguousarray(emb)).to(dev)
            m = torch.from_numpy(mask).to(dev)
            self.bits = pack_bits_torch(m)
            self.queries = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to(dev)
            self.lo, self.n_sel, self.n_sel_total = 0, int(mask.sum()), int(mask.sum())
        elif cfg.get("host"):
            # this rank's 1/8 shard (ranks 0..7 hold shards 0..7), generated on
            # the device chunk by chunk and parked in pinned host memory
            n_sh = cfg["n"] // cfg["shards"]
            self.lo = (rank % cfg["shards"]) * n_sh
            t0 = time.time()
            host = torch.empty((n_sh, cfg["d"]), dtype=torch.float32).pin_memory()
            chunk = 1 << 20
            centers = None
            for a in range(0, n_sh, chunk):
                b = min(n_sh, a + chunk)
                part, centers = _device_slice(cfg["n"], cfg["d"], self.lo + a, self.lo + b, dev)
                host[a:b].copy_(part)
                del part
            g = torch.Generator(device=dev)
            g.manual_seed(4242)
            mask = torch.rand(cfg["n"], generator=g, device=dev)[self.lo:self.lo + n_sh] < cfg["sel"]
            self.bits = pack_bits_torch(mask.contiguous())
            from paper_2605_15957_b200 import synth
            self.queries = synth.device_queries(centers, self.nq, seed=7)
            self.n_sel = self.n_sel_total = int(mask.sum())
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            log(f"[rank {rank}] cfg5 shard {n_sh} x {cfg['d']} in pinned host memory ({time.time() - t0:.1f}s)")
            self.host_data = host
            self.col = vs.EmbeddingColumn.host_resident(host)
            self.h2d_peak = _pinned_h2d_gbs(dev)
            data = None
        else:
            W = build_cfg2(rank, world, cfg)
            data, self.bits, self.queries = W["data"], W["bits"], W["queries"]
            self.lo, self.n_sel, self.n_sel_total = W["lo"], W["n_sel"], W["n_sel_total"]
        if data is not None:
            self.col = vs.EmbeddingColumn.from_device(data)
        nq, k = self.nq, self.k
        self.out_dev = (torch.empty((nq, k), dtype=torch.int64, device=dev),
                        torch.empty((nq, k), dtype=torch.float64, device=dev),
                        torch.empty((nq,), dtype=torch.int32, device=dev))
        self.q_host = self.queries.cpu().pin_memory()
        self.bits_host = self.bits.cpu().pin_memory()
        self.out_host = tuple(_pinned_like(t) for t in self.out_dev)
        self.sharded = world > 1 and not self.replicas

    def _search(self, q, bits, out):
        from paper_2605_15957_b200.vecindex import enn_search_raw
        enn_search_raw(q, self.col, self.k, "squared_l2", row_filter=bits, id_offset=self.lo, out=out)

    def _exchange(self):
        from paper_2605_15957_b200.distributed import all_gather_topk, gpu_merge
        gi, gd, gc = all_gather_topk(*self.out_dev)
        return gpu_merge(gi, gd, gc, self.k, "squared_l2")

    def _two_phase(self, q, bits):
        """Row shards with the two-phase protocol (distributed.two_phase_search):
        one all-reduce of the shard-local k-th keys, phase B on each shard's
        candidates under the global bound, all-gather + merge kernel."""
        from paper_2605_15957_b200.distributed import ShardSearch, TorchComm, two_phase_search
        if not hasattr(self, "_shard"):
            self._shard = ShardSearch(self.col)
            self._comm = TorchComm()
        return two_phase_search(self._shard, self._comm, q, self.k, "squared_l2", row_filter=bits,
                                id_offset=self.lo)

    def step_device(self):
        if self.sharded and not self.cfg.get("host"):
            self.out_dev = self._two_phase(self.queries, self.bits)
            return
        self._search(self.queries, self.bits, self.out_dev)
        if self.sharded:
            self._exchange()

    def step_e2e(self):
        if not self.sharded:
            self._search(self.q_host, self.bits_host, self.out_host)
            return
        if not self.cfg.get("host"):
            # host queries and bitmap in; the global result back to the host
            q = self.q_host.to(self.dev, non_blocking=True)
            b = self.bits_host.to(self.dev, non_blocking=True)
            for h, t in zip(self.out_host, self._two_phase(q, b)):
                h.copy_(t)
            return
        self._search(self.q_host, self.bits_host, self.out_dev)
        for h, t in zip(self.out_host, self._exchange()):
            h.copy_(t)

    def check(self):
        ids, dd, cc = self.out_dev
        n_sel = self.n_sel_total if self.sharded else self.n_sel
        assert int(cc.min()) == min(self.k, n_sel), "short result rows"
        assert bool((dd[:, 1:] >= dd[:, :-1]).all()), "distances not sorted"
        if self.world == 1:
            self._check_oracle()

    def _check_oracle(self):
        """Two sampled queries (first and last of the batch) bit-exact against
        the oracle over the host copy of the selected rows (checker only,
        outside the timed region; oracle.enn_pruned = enn_search's arithmetic)."""
        import torch

        from oracle import sqlvs_oracle as O
        qi = np.array([0, self.nq - 1])
        if self.cfg.get("host"):
            mask = np.unpackbits(self.bits.cpu().numpy().view(np.uint8), bitorder="little")[:self.host_data.shape[0]]
            rows = np.flatnonzero(mask)
            xs = self.host_data.numpy()[rows]
        elif self.replicas:
            emb, mask, _ = self.host_sample
            rows = np.flatnonzero(mask)
            xs = emb[rows]
        else:
            m = torch.from_numpy(np.unpackbits(self.bits.cpu().numpy().view(np.uint8), bitorder="little")
                                 [:self.col.count].astype(bool)).to(self.dev)
            r = torch.nonzero(m).flatten()
            xs = self.col._dev_tensor[r].float().cpu().numpy()
            rows = r.cpu().numpy()
        q = self.queries[torch.from_numpy(qi).to(self.dev)].cpu().numpy()
        ref = O.enn_pruned(q, xs, self.k, "squared_l2", row_ids=rows + self.lo)
        ids, dd, cc = (t.cpu().numpy() for t in self.out_dev)
        for j, i in enumerate(qi):
            want_i, want_d = ref.per_query(j)
            c = int(cc[i])
            if not (np.array_equal(ids[i, :c], want_i) and np.array_equal(dd[i, :c], want_d)):
                raise SystemExit(f"PARITY FAILURE: query {i} differs from the oracle")
        log(f"check: queries {qi.tolist()} bit-exact vs the oracle")

    def io_bytes(self):
        h2d = self.q_host.numel() * 4 + self.bits_host.numel() * 4
        d2h = sum(t.numel() * t.element_size() for t in self.out_host)
        return h2d, d2h

    def units_per_step(self):
        return self.nq * (self.world if self.replicas else 1)

    def scaling(self):
        return "weak" if (self.replicas or self.cfg.get("host")) else "strong"

    def roofline(self, kt, steps, ctx, N):
        tc = "tcgen05_bf16" if os.environ.get("VS_TC_BF16") == "1" else "tcgen05_fp16"
        self.kernel_name = {1: "simt_fp32", 2: tc, 3: "wide"}.get(ctx.stats()[N.STAT_LAST_ENN_KERNEL], "?")
        if self.cfg.get("host"):
            # streamed variant: the bound is the PCIe transfer of the selected rows
            byts = float(self.n_sel) * self.d * 4
            ms = self.last_ms_step
            achieved = byts / (ms / 1e3) / 1e9
            return {"bound": "pcie", "kernel": "whole search (selected-row gather over PCIe + tcgen05 scan)",
                    "achieved": round(achieved, 2), "peak": round(self.h2d_peak, 2), "unit": "GB/s",
                    "frac": round(achieved / self.h2d_peak, 4),
                    "peak_source": "measured in this run: pinned host->device copy of 1 GiB",
                    "algorithmic_bytes_per_step": byts, "traffic": None}
        peaks = measured_peaks()
        scan_ns, scan_n = kt["enn_scan"]
        flops = 2.0 * self.nq * self.n_sel * self.d
        achieved = flops / (scan_ns / max(scan_n, 1) / 1e9) / 1e12 if scan_n else None
        peak = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
        kern = self.kernel_name
        traffic = _traffic(f"cfg{self.cfg['id']}:{kern}")
        return {"bound": "tensor", "kernel": f"enn_scan ({kern})",
                "achieved": round(achieved, 2) if achieved else None, "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (of measured; dense fp16 runs at the "
                               "bf16 rate)",
                "algorithmic_flops_per_launch": flops, "traffic": traffic}

    def config(self):
        c = self.cfg
        par = ("replicas x%d (query batches independent)" % self.world if self.replicas else
               f"row-shard x{self.world}: two-phase (all-reduce MIN of shard k-th keys, bounded "
               f"re-rank) + all-gather/merge kernel") if self.world > 1 else "single GPU"
        if c.get("host"):
            par = f"{self.world} of {c['shards']} row shards (one per GPU), host-resident, allgather/merge"
        n_rows = c["n"] // c["shards"] * self.world if c.get("host") else c["n"]
        return {"workload": c["name"], "n_rows": n_rows, "dim": self.d, "queries": self.nq, "k": self.k,
                "selectivity": c["sel"], "n_selected": self.n_sel_total, "parallelism": par,
                "l2_flush": ("inputs larger than L2 (41 GB collection vs 126 MB L2)" if c["id"] == 2 else
                             "inputs in host memory (38.4 GB shard), streamed every step" if c["id"] == 5 else
                             "none: 16.5 MB selected working set is L2-resident (latency-bound config)"),
                "phase_a_kernel": getattr(self, "kernel_name", "?")}

    def dtype(self):
        kern = getattr(self, "kernel_name", "")
        cand = ("fp16 (power-of-two scaled) tcgen05 candidates" if kern == "tcgen05_fp16" else
                "bf16 tcgen05 candidates" if kern == "tcgen05_bf16" else "fp32 SIMT candidates")
        return "f32 storage; " + cand + "; f64 exact re-rank"

    def extras(self, ctx, N):
        st = ctx.stats()
        ex = {"survivors_per_query": round(st[N.STAT_SURVIVORS] / self.nq, 2),
              "overflow_requeries_total": int(st[N.STAT_OVERFLOW_QUERIES])}
        if self.cfg["id"] == 1:
            ex["gpu_filter_ms"] = self._gpu_filter_ms()
        return ex

    def _gpu_filter_ms(self):
        """Config 1's relational filter built on the GPU from the raw columns:
        isin(rv_partkey, part[p_size <= 5].p_partkey) as a packed bitmap
        (predicate.compare + predicate.isin; checked against the host mask)."""
        import torch

        from paper_2605_15957_b200 import predicate as P
        from paper_2605_15957_b200 import synth
        spec = synth.Spec(sf=0.1, d_r=384, d_i=384, seed=42)
        pk = torch.from_numpy(synth.review_partkeys(spec)[:self.cfg["n"]].astype(np.int64)).to(self.dev)
        psize = torch.from_numpy(synth.part_sizes(spec).astype(np.int64)).to(self.dev)
        pkeys = torch.arange(1, psize.numel() + 1, dtype=torch.int64, device=self.dev)

        def run():
            small = pkeys[torch.from_numpy(synth.unpack_bitmap(
                P.compare(psize, "<=", 5).cpu().numpy().view(np.uint32), psize.numel())).to(self.dev)]
            return P.isin(pk, small)
        bits = run()
        assert torch.equal(bits, self.bits), "GPU filter differs from the reference mask"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            run()
        torch.cuda.synchronize()
        return round((time.perf_counter() - t0) / 20 * 1e3, 3)

    def cpu_baseline(self, args):
        if self.cfg["id"] == 1:
            return time_cpu_cfg1(self.host_sample, self.k, args.cpu_budget)
        cfg = dict(self.cfg)
        if cfg.get("host"):
            cfg["n"] = cfg["n"] // cfg["shards"]   # the same per-GPU shard the GPU arm searches
        qps_cpu, sample, cores = time_cpu_reference(cfg, budget_s=args.cpu_budget, processes=1)
        return {"value": round(qps_cpu, 6), "unit": "queries/s", "cores": cores, "kind": "port",
                "sample": sample}


def _pinned_h2d_gbs(dev):
    import torch
    a = torch.empty(1 << 28, dtype=torch.float32).pin_memory()
    b = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    b.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        b.copy_(a, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 3 * a.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9


def time_cpu_cfg1(sample, k, budget_s):
    """The reference composition on the real config-1 inputs (no
    extrapolation): gather the filtered rows, then enn_search per query."""
    from oracle import sqlvs_oracle as O
    emb, mask, q = sample
    rows = np.flatnonzero(mask)
    xs = np.ascontiguousarray(emb[rows])
    t0 = time.perf_counter()
    done = 0
    while done < len(q) and time.perf_counter() - t0 < budget_s:
        O.enn_search(q[done:done + 8], xs, k, row_ids=rows)
        done += min(8, len(q) - done)
    el = time.perf_counter() - t0
    return {"value": round(done / el, 4), "unit": "queries/s", "cores": 1, "kind": "port",
            "sample": f"{done} of {len(q)} config-1 queries over the {rows.size} selected rows in {el:.1f}s"}


class IvfWorkload:
    """Config 3: filtered IVF-Flat search over the list-contiguous (owning)
    layout. The index is built on the GPU (vs_ivf_build, the reference's
    k-means semantics); under torchrun, lists are LPT-assigned to ranks and
    the per-rank top-k are all-gathered and merged."""

    def __init__(self, args, cfg, rank, world, dev):
        import torch

        import paper_2605_15957_b200 as vs
        from paper_2605_15957_b200 import synth
        from paper_2605_15957_b200.distributed import lpt_assign
        self.cfg, self.rank, self.world, self.dev = cfg, rank, world, dev
        self.k, self.nq, self.d, self.nprobe = cfg["k"], cfg["q"], cfg["d"], cfg["nprobe"]
        n, d = cfg["n"], cfg["d"]
        self.bf16 = bool(cfg.get("bf16"))
        self.index_dtype = "bf16" if self.bf16 else "f32"
        t0 = time.time()
        data, centers = (_device_slice_bf16 if self.bf16 else _device_slice)(n, d, 0, n, dev)
        if cfg["sel"] is not None:
            g = torch.Generator(device=dev)
            g.manual_seed(4243)
            mask = torch.rand(n, generator=g, device=dev) < cfg["sel"]
            self.bits = pack_bits_torch(mask)
        else:
            mask, self.bits = None, None
        self.queries = synth.device_queries(centers, self.nq, seed=7)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        log(f"[rank {rank}] generated {n} x {d} ({'bf16' if self.bf16 else 'f32'}) in {time.time() - t0:.1f}s")
        t0 = time.time()
        col = vs.EmbeddingColumn.from_device(data)
        from paper_2605_15957_b200 import _native as N
        ties0 = N.Context.get().stats()[N.STAT_NEAR_TIES]
        self.index = vs.IvfIndex.build(col, cfg["nlist"], seed=0, max_iters=cfg.get("iters", 20))
        torch.cuda.synchronize()
        self.build_s = time.time() - t0
        self.build_ties = int(N.Context.get().stats()[N.STAT_NEAR_TIES] - ties0)
        log(f"[rank {rank}] IVF build nlist={cfg['nlist']} in {self.build_s:.1f}s "
            f"({self.build_ties} near-tie rows re-checked exactly over all iterations)")
        sizes = np.array([len(p) for p in self.index.partitions], np.int64)
        self.list_sizes = sizes
        self.owned = None
        if world > 1:
            owner = lpt_assign(sizes, world)
            self.owned = (owner == rank).astype(np.uint8)
        # host copies for the roofline bytes and the CPU reference sample
        if mask is not None:
            self.mask_host = mask.cpu().numpy()
            ids_host = np.concatenate(self.index.partitions)
            self.sel_per_list = np.add.reduceat(self.mask_host[ids_host].astype(np.int64),
                                                np.r_[0, np.cumsum(sizes)[:-1]]) if n else sizes * 0
            self.sel_per_list[sizes == 0] = 0
        else:
            self.mask_host = None
            self.sel_per_list = sizes
        # CPU sample: the first queries' probed lists, gathered before the
        # base collection is released (the owning index keeps its own payload)
        self.cpu_q = self.queries[:cfg.get("cpu_queries", 16)].cpu().numpy()
        _, _, _, probes, _ = self.index.search_raw(self.cpu_q, self.k, self.nprobe, row_filter=self.bits,
                                                   list_owned=self.owned)
        self.cpu_lists = {int(c): data[torch.from_numpy(self.index.partitions[int(c)]).to(dev)].float().cpu().numpy()
                          for c in np.unique(probes)}
        self.cpu_probes = probes
        del col, data
        torch.cuda.empty_cache()
        nq, k = self.nq, self.k
        self.out_dev = (torch.empty((nq, k), dtype=torch.int64, device=dev),
                        torch.empty((nq, k), dtype=torch.float64, device=dev),
                        torch.empty((nq,), dtype=torch.int32, device=dev))
        self.q_host = self.queries.cpu().pin_memory()
        self.bits_host = self.bits.cpu().pin_memory() if self.bits is not None else None
        self.out_host = tuple(_pinned_like(t) for t in self.out_dev)
        self.n_sel_total = int(mask.sum()) if mask is not None else n

    def _search(self, q, bits, out, want_probes=False):
        return self.index.search_raw(q, self.k, self.nprobe, row_filter=bits, out=out,
                                     list_owned=self.owned, want_probes=want_probes)

    def _exchange(self):
        from paper_2605_15957_b200.distributed import all_gather_topk, gpu_merge
        gi, gd, gc = all_gather_topk(*self.out_dev)
        return gpu_merge(gi, gd, gc, self.k, "squared_l2")

    def step_device(self):
        if self.world > 1:
            # coarse quantizer split by queries, probes all-gathered, owned
            # lists scanned, top-k all-gathered + merged (distributed.ivf_sharded_search)
            from paper_2605_15957_b200.distributed import ivf_sharded_search
            self.out_dev = ivf_sharded_search(self.index, self.queries, self.k, self.nprobe,
                                              row_filter=self.bits, list_owned=self.owned)
            return
        self._search(self.queries, self.bits, self.out_dev)

    def step_e2e(self):
        if self.world == 1:
            self._search(self.q_host, self.bits_host, self.out_host)
            return
        from paper_2605_15957_b200.distributed import ivf_sharded_search
        q = self.q_host.to(self.dev, non_blocking=True)
        b = self.bits_host.to(self.dev, non_blocking=True) if self.bits_host is not None else None
        res = ivf_sharded_search(self.index, q, self.k, self.nprobe, row_filter=b, list_owned=self.owned)
        for h, t in zip(self.out_host, res):
            h.copy_(t)

    def check(self):
        ids, dd, cc = self.out_dev
        assert bool(((dd[:, 1:] >= dd[:, :-1]) | dd[:, 1:].isnan()).all()), "distances not sorted"
        if self.world > 1:
            return
        # two sampled queries (their probed lists were gathered at setup) bit-exact
        # against the oracle's IVF search (checker only, outside the timed region)
        from oracle import sqlvs_oracle as O
        qi = [0, len(self.cpu_q) - 1]
        res = O.ivf_search(self.cpu_q[qi], self.index.centroids, self.index.partitions, lambda c: self.cpu_lists[c],
                           self.nprobe, self.k, mask=self.mask_host)
        ids, dd, cc = (t.cpu().numpy() for t in self.out_dev)
        for j, i in enumerate(qi):
            want_i, want_d = res.per_query(j)
            c = int(cc[i])
            if not (np.array_equal(res.probes[j], self.cpu_probes[i]) and np.array_equal(ids[i, :c], want_i)
                    and np.array_equal(dd[i, :c], want_d)):
                raise SystemExit(f"PARITY FAILURE: query {i} differs from the oracle")
        log(f"check: queries {qi} (probes, ids, distances) bit-exact vs the oracle")

    def io_bytes(self):
        h2d = self.q_host.numel() * 4 + (self.bits_host.numel() * 4 if self.bits_host is not None else 0)
        d2h = sum(t.numel() * t.element_size() for t in self.out_host)
        return h2d, d2h

    def units_per_step(self):
        return self.nq

    def scaling(self):
        return "strong"

    def scan_bytes(self):
        """Algorithmic bytes of one IVF list-scan launch:
        over the unique lists probed by the batch (and owned by this rank),
        the list's permuted-bitmap bits plus its selected rows' payload."""
        _, _, _, probes, _ = self._search(self.q_host, self.bits_host, None, want_probes=True)
        uniq = np.unique(probes)
        if self.owned is not None:
            uniq = uniq[self.owned[uniq] == 1]
        s = 4 if self.index_dtype == "f32" else 2
        self.unique_lists = int(uniq.size)
        # probe skew: lists probed by more queries than one query tile (128)
        # are scanned once per tile
        pairs = np.bincount(np.asarray(probes).ravel(), minlength=len(self.list_sizes))
        passes = np.ceil(pairs[uniq] / 128.0)
        rows = self.sel_per_list[uniq]
        self.list_pairs = {"mean": round(float(pairs[uniq].mean()), 1), "p99": int(np.percentile(pairs[uniq], 99)),
                           "max": int(pairs.max()),
                           "row_passes": round(float(np.sum(passes * rows) / max(np.sum(rows), 1)), 4)}
        bitmap = self.list_sizes[uniq] / 8.0 if self.bits is not None else 0.0
        return float(np.sum(bitmap + self.sel_per_list[uniq] * self.d * s))

    def roofline(self, kt, steps, ctx, N):
        peaks = measured_peaks()
        ns, n = kt["ivf_scan"]
        byts = self.scan_bytes()
        achieved = byts / (ns / max(n, 1) / 1e9) / 1e9 if n else None
        peak = peaks["hbm_gbs"]
        self.kt = kt
        return {"bound": "hbm", "kernel": "ivf_scan (list scan, filtered)",
                "achieved": round(achieved, 2) if achieved else None, "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic_bytes_per_launch": byts,
                "traffic": _traffic(f"cfg{self.cfg['id']}:ivf_scan")}

    def config(self):
        c = self.cfg
        return {"workload": c["name"], "n_rows": c["n"], "dim": self.d, "queries": self.nq, "k": self.k,
                "nlist": c["nlist"], "nprobe": self.nprobe, "selectivity": c["sel"],
                "n_selected": self.n_sel_total, "unique_probed_lists": getattr(self, "unique_lists", None),
                "pairs_per_list": getattr(self, "list_pairs", None),
                "build_s": round(self.build_s, 2),
                "build_near_tie_rechecks": self.build_ties,
                "list_rows": {"mean": round(float(np.mean(self.list_sizes)), 1),
                              "p99": int(np.percentile(self.list_sizes, 99)),
                              "max": int(np.max(self.list_sizes))},
                "parallelism": (f"list-shard (LPT) x{self.world}: coarse split by queries + probe all-gather, "
                                f"owned-list scans, top-k all-gather/merge") if self.world > 1 else "single GPU",
                "l2_flush": "inputs larger than L2 (41 GB payload vs 126 MB L2)"}

    def dtype(self):
        return "f32 storage; fp32 list scan; f64 exact re-rank"

    def extras(self, ctx, N):
        import torch
        if self.world > 1:
            return {"overflow_requeries_total": int(ctx.stats()[N.STAT_OVERFLOW_QUERIES])}
        # survivors of the last phase B (the IVF re-rank of the timed batch)
        surv = round(ctx.stats()[N.STAT_SURVIVORS] / self.nq, 2)
        lat = {}
        for qn in (1, 100):
            q = self.queries[:qn].contiguous()
            out = tuple(t[:qn].contiguous() for t in self.out_dev)
            for _ in range(2):
                self._search(q, self.bits, out)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 20
            for _ in range(reps):
                self._search(q, self.bits, out)
            torch.cuda.synchronize()
            lat[f"Q={qn}"] = round((time.perf_counter() - t0) / reps * 1e3, 3)
        return {"batch_latency_ms": lat, "ivf_survivors_per_query": surv,
                "overflow_requeries_total": int(ctx.stats()[N.STAT_OVERFLOW_QUERIES])}

    def cpu_baseline(self, args):
        """The reference IVF search path (oracle port of vecindex.py:230-258,
        filtered) on the first queries, over the real centroids and the real
        probed lists; also checks our results for those queries bit-exactly."""
        from oracle import sqlvs_oracle as O
        t0 = time.perf_counter()
        done, first = 0, None
        try:
            while done < len(self.cpu_q) and time.perf_counter() - t0 < args.cpu_budget:
                res = O.ivf_search(self.cpu_q[done:done + 1], self.index.centroids, self.index.partitions,
                                   lambda c: self.cpu_lists[c], self.nprobe, self.k, mask=self.mask_host)
                if done == 0:
                    first = res
                done += 1
        except KeyError as e:   # the oracle probed a list our probes did not: parity failure
            return {"value": None, "unit": "queries/s", "cores": 1, "kind": "port",
                    "sample": f"ABORTED: oracle probe {e} not among our probed lists (probe parity failure)"}
        el = time.perf_counter() - t0
        ids, dist, cnt, probes, _ = self.index.search_raw(self.cpu_q[:1], self.k, self.nprobe,
                                                          row_filter=self.bits_host, list_owned=self.owned)
        parity = bool(np.array_equal(first.probes[0], probes[0]) and
                      np.array_equal(first.data_row, ids[0][:cnt[0]]) and
                      np.array_equal(first.distance, dist[0][:cnt[0]])) if self.world == 1 else None
        return {"value": round(done / el, 4), "unit": "queries/s", "cores": 1, "kind": "port",
                "sample": f"{done} queries, full reference IVF path (fp64 coarse over {self.cfg['nlist']} "
                          f"centroids + probed-list concat/filter/score) in {el:.1f}s; "
                          f"query-0 bit-exact vs ours: {parity}"}


class IvfBf16Workload(IvfWorkload):
    """Config 4: IVF-Flat over 50M x 768 bf16 embeddings (76.8 GB), built on
    the GPU over the whole collection with the reference's k-means semantics
    (the payload copy is the list-contiguous layout; the generated column is
    released after the build), searched with the list-major tcgen05 scan."""

    def roofline(self, kt, steps, ctx, N):
        r = super().roofline(kt, steps, ctx, N)
        r["kernel"] = "ivf_scan (tcgen05 list-major, bf16 payload)"
        return r

    def config(self):
        c = super().config()
        c.update(selectivity=None, l2_flush="inputs larger than L2 (76.8 GB payload vs 126 MB L2)")
        return c

    def dtype(self):
        return "bf16 storage; bf16 tcgen05 list scan (fp32 accumulate); f64 exact re-rank"


def _traffic(key):
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        return json.loads(tp.read_text()).get(key)
    return None


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2605_15957_b200 import _native as N

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: VS_BENCH_ONE_GPU=1 puts every rank on cuda:0 and talks gloo,
    # which exercises the N > 1 code path on a one-GPU box (never for numbers)
    one_gpu = os.environ.get("VS_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    H = Harness(world, dev)
    wl = (IvfBf16Workload if cfg.get("bf16") else IvfWorkload if "nlist" in cfg else ExactWorkload)(
        args, cfg, rank, world, dev)
    ctx = N.Context.get(local)
    if args.cand_slack:
        ctx.set_option(N.OPT_CAND_SLACK, args.cand_slack)

    log(f"[rank {rank}] warmup {args.warmup}")
    for _ in range(args.warmup):
        wl.step_device()
    torch.cuda.synchronize()
    if args.warmup > 0:
        wl.check()

    launches0 = ctx.stats()[N.STAT_LAUNCHES]
    ctx.set_option(N.OPT_TIMING, 1)
    ctx.kernel_times(reset=True)
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include timed/ selects these launches
    with ClockSampler(local) as clk:
        ms = H.timed(wl.step_device, args.steps)
    torch.cuda.nvtx.range_pop()
    kt = ctx.kernel_times(reset=True)
    ctx.set_option(N.OPT_TIMING, 0)
    launches = ctx.stats()[N.STAT_LAUNCHES] - launches0
    extras = wl.extras(ctx, N)
    for _ in range(2):
        wl.step_e2e()
    ctx.set_option(N.OPT_TIMING, 1)
    ctx.kernel_times(reset=True)
    t_host = time.perf_counter()
    ms_e2e = H.timed(wl.step_e2e, args.steps)
    t_host = (time.perf_counter() - t_host) * 1e3
    kt_e2e = ctx.kernel_times(reset=True)
    ctx.set_option(N.OPT_TIMING, 0)

    units = wl.units_per_step()
    wl.last_ms_step = ms / args.steps
    qps = units * args.steps / (ms / 1e3)
    qps_e2e = units * args.steps / (ms_e2e / 1e3)
    roof = wl.roofline(kt, args.steps, ctx, N)
    result = None
    if rank == 0:
        h2d, d2h = wl.io_bytes()
        result = {
            "metric": "filtered top-k queries/sec",
            "value": round(qps, 3),
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3),
            "higher_is_better": True,
            "scaling": wl.scaling(),
            "vs_baseline": None,
            "dtype": wl.dtype(),
            "data": "synthetic (Vec-H mixture law; seeded bitmap)",
            "config": wl.config(),
            "e2e": {"value": round(qps_e2e, 3), "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "kernel_ms_per_step": {c: round(v[0] / 1e6 / args.steps, 3) for c, v in kt.items() if v[1]},
            "e2e_kernel_ms_per_step": {c: round(v[0] / 1e6 / args.steps, 3) for c, v in kt_e2e.items() if v[1]},
            "e2e_host_ms_per_step": round(t_host / args.steps, 3),
            "roofline": roof,
            "clocks": clk.summary(),
        }
        result.update(extras)
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = wl.cpu_baseline(args)
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
        qps, sample, _ = time_cpu_reference(cfg, budget_s=args.ref_budget, processes=procs, use_reference=True)
        if i >= args.warmup:
            vals.append(qps)
    v = statistics.median(vals)
    kind = "reference" if _SAMPLE.get("ref") is not None else "port"
    sample += ("; the unmodified reference sqlvs.vecindex.enn_search (oracle/_ref)" if kind == "reference"
               else "; the oracle port of enn_search (oracle/_ref absent)")
    print(json.dumps({
        "impl": "reference", "metric": "filtered top-k queries/sec", "value": round(v, 6),
        "unit": "queries/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (Vec-H mixture law, host sample)",
        "config": {"workload": cfg["name"]},
        "cpu_baseline": {"value": round(v, 6), "unit": "queries/s", "cores": procs, "kind": kind,
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
    ap.add_argument("--cand-slack", type=int, default=0, help="VS_OPT_CAND_SLACK (candidate buffer x2^s)")
    ap.add_argument("--n-rows", type=int, default=0,
                    help="code-path runs only (e.g. the N>1 path on one GPU): a smaller collection; "
                         "never used for reported numbers")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.n_rows:
        cfg.update(n=args.n_rows, name=cfg["name"] + f" [CODE-PATH RUN: {args.n_rows} rows]")
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
