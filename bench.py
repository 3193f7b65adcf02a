#!/usr/bin/env python
"""Benchmark of the k=1 fingerprint-filtered query x dictionary scan.

Metric (BASELINE.json:2): logical query x word comparisons per second,
Q * N per batch (the reference's pair denominator, bench.hpp:157-161), whole
job over all GPUs.  Default workload = config 5 (BASELINE.json:11, the
configuration the metric is quoted on "at 1/2/4/8 B200"): 64,000,000 uniform
a-z words, L~U[4,16], one batch of 1,000,000 queries (50% one edit, 50%
random), cell 0 = occurrence-16 fingerprints, Hamming, k = 1, per-query
QueryStats on (run_pass collects them, bench.hpp:80-90).  One step = one
batch through the scan.  Letters are selected over the whole 64M-word
dictionary and query sources are drawn from all of it.

Scaling is STRONG for config 5 (BASELINE: one 64M-word dictionary "sharded
evenly across 8xB200"): with N GPUs each owns 64M/N words (contiguous
input-order id ranges) and scans the same 1M queries.  Other configs run
weak scaling (each GPU holds a copy-sized shard of the config's stream).

  --gpus N without torchrun: ONE process drives N GPUs (devices 0..N-1)
      through GpuFingerprintedDictionary(devices=...); libfpg.so gathers the
      shard rows on the host inside the e2e call.  Fails loudly if fewer
      than N devices exist (FPG_BENCH_DEVICES="0,0" overrides, for tests).
  torchrun --nproc-per-node N ... --gpus N: one process per GPU (asserted
      WORLD_SIZE == N); rank r owns shard r; the e2e step gathers the ranks'
      device-resident CSRs to rank 0 over NCCL and merges them there on the
      GPU (sharding.query_batch_distributed).

  value  device-resident: inputs already in HBM, CUDA-event time of
         fpg_batch_run (K1 on the queries, K2, K4), max over shards / ranks
  e2e    through the public API with pinned host buffers: H2D of the
         queries, scan, gather + merge of the shards, D2H of the CSR (+
         QueryStats on one process), wall time, max over ranks

--impl reference runs the reference's own CPU implementation
(oracle/_ref/libfpref.so: /root/reference headers, FingerprintedDictionary::
query_into) on all host threads over a bounded query sample of the same
workload, on rank 0 only; libfpg.so is never loaded in that process.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "k=1 query x word comparisons/s (logical Q*N)"
POPC_PER_CLK_PER_SM = 16  # measured: tools/microbench/intpipe.cu (profiles/r01_phase0.txt)
L2_NOTE = "flushed between timed steps (256 MB write > 126 MB L2)"


def alu_peak():
    """(LOP3 thread-ops per clk per SM, basis) from the committed B200
    microbenchmark (tools/microbench/alupipe.cu -> profiles/alu_peak.json)."""
    try:
        rec = json.loads((ROOT / "profiles" / "alu_peak.json").read_text())
        return float(rec["lop3_per_clk_per_sm"]), rec["basis"]
    except (OSError, ValueError, KeyError):
        return 64.0, "unmeasured: 16 lanes/clk/SMSP (B300_MICROARCH.md pipe rates)"


def imad_peak() -> float:
    """IMAD thread-ops per clk per SM (FMA pipe), same microbenchmark."""
    try:
        return float(json.loads((ROOT / "profiles" / "alu_peak.json").read_text())["imad_per_clk_per_sm"])
    except (OSError, ValueError, KeyError):
        return 64.0


def imads_per_comparison(scheme, sig_fields: int, exact: bool = False) -> float:
    """IMAD per comparison (the query XOR of every plane, FMA pipe): one per
    plane and 32-word slab; even field widths fold their last plane into the
    field OR instead (fpg_slice.cuh)."""
    if exact:
        return X_BITS * X_LEN / 32.0
    v, w = scheme.variant().name, scheme.width()
    fw = scheme.bits_per_count() if v == "Count" else scheme.bits_per_position() if v == "Position" else 1
    extra = w % fw if v == "Position" else 0
    nf = (w - extra) // fw
    planes = nf * (fw - 1 if fw % 2 == 0 else fw) + extra + sig_fields
    return planes / 32.0


X_LEN, X_BITS = 6, 5  # the exact Hamming path of short words (fpg_kernels.cuh kXLen / kXBits)


def ops_per_comparison(scheme, sig_fields: int, exact: bool = False) -> float:
    """LOP3 per comparison of the bit-sliced test (fpg_slice.cuh): per 32-word
    slab, the ORs folding a multi-bit field's planes (1 for 2-3 bits, 2 for 4
    bits), then the carry-save counter: 6 per four field bits plus one
    fours-carry OR per two such quads, 4 per remaining pair or single, counted
    separately over the scheme fields and the sig' fields (one-bit), plus 1
    for the reject mask."""
    v, w = scheme.variant().name, scheme.width()
    if v == "Count":
        fw, extra = scheme.bits_per_count(), 0
    elif v == "Position":
        fw = scheme.bits_per_position()
        extra = w % fw
    else:
        fw, extra = 1, 0
    nf = (w - extra) // fw

    def csa(n: int) -> int:  # 6 per quad + one carry OR per two quads, 4 per pair / single
        q4 = n // 4
        return 6 * q4 + (q4 + 1) // 2 + 4 * ((n % 4 + 1) // 2)

    ors = nf * (0 if fw == 1 else 1 if fw <= 3 else 2)
    if exact:
        # position fields: a 5-plane OR (2 LOP3) each, their own counter and the
        # pass mask (the scheme fields are not counted there any more: QueryStats
        # come from the fingerprint histograms)
        return (2 * X_LEN + csa(X_LEN) + 1) / 32.0
    return (ors + csa(nf + extra) + csa(sig_fields) + 1) / 32.0


def hbm_peak():
    """(GB/s, basis): the driver-measured copy bandwidth of this pool's B200s
    (MEASURED_PEAKS.json), else the B200_PROFILING.md fallback."""
    try:
        rec = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(rec["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver: torch copy, read + write bytes)"
    except (OSError, ValueError, KeyError):
        return 7700.0, "fallback: nominal B200 HBM3e (MEASURED_PEAKS.json absent)"


def construction_roofline(d) -> dict:
    """HBM roofline of dictionary construction (shard 0): per stage, the
    CUDA-event time and algorithmic bytes from fpg_dict_build_profile."""
    peak, basis = hbm_peak()
    stages = []
    for st in d.build_profile(0):
        gbs = st["bytes"] / (st["ms"] * 1e6) if st["ms"] > 0 else None
        stages.append({"stage": st["name"], "ms": st["ms"], "algorithmic_bytes": st["bytes"], "gbs": gbs,
                       "frac": gbs / peak if gbs else None})
    return {"bound": "hbm", "peak_gbs": peak, "peak_basis": basis, "stages": stages,
            "note": "cub_radix_sort is CUB's onesweep (library); bytes = one key+value read+write per 8-bit pass"}


def profiled_traffic(workload: str, cell: str):
    """DRAM bytes of one K2 launch from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_summary.py traffic)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        rec = json.loads(p.read_text()).get(f"{workload} {cell}")
    except (OSError, ValueError):
        return None
    return rec["dram_bytes"] if rec else None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--cell", type=int, default=0, help="index into corpus.CELLS[config]")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs)")
    return ap.parse_args()


class Clocks:
    """NVML sampling (every 10 ms, background thread) of SM clocks and clock
    event (throttle) reasons, kept only while the timed region is open."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index, self.samples, self.active, self.stop_flag = index, [], False, False
        self.max_mhz, self.err = None, None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # no NVML: report it, never guess
            self.nv, self.err = None, f"nvml unavailable: {e}"

    def _loop(self):
        while not self.stop_flag:
            if self.active:
                try:
                    sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                    rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((float(sm), int(rs)))
                except Exception as e:
                    self.err = str(e)
            time.sleep(0.01)

    def start(self):
        if self.nv:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()

    def open(self):
        self.active = True

    def close(self):
        self.active = False

    def stop(self) -> dict:
        self.stop_flag = True
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [self.err or "no samples"]}
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, 10 ms"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Workload:
    """The config's whole dictionary and query batch (seeded generators), the
    scheme with letters chosen over the whole dictionary, and the shard this
    process owns."""

    def __init__(self, cfg: int, cell: int, parts: int = 1, part: int = 0):
        from paper_1711_08475_b200.corpus import CELLS, CONFIGS, generate_dictionary, generate_queries, make_scheme
        from paper_1711_08475_b200.sharding import shard_bounds, shard_of

        self.cfg, self.cell, self.c = cfg, cell, CONFIGS[cfg]
        self.strong = cfg == 5  # config 5: one dictionary split over the GPUs
        n_all = self.c.n_words if self.strong else self.c.n_words * parts
        t0 = time.perf_counter()
        self.blob, self.offs = generate_dictionary(cfg, n=n_all)
        self.qblob, self.qoffs = generate_queries(cfg, self.blob, self.offs, nq=self.c.n_queries)
        variant, width, b, p, self.metric = CELLS[cfg][cell]
        self.scheme = make_scheme(self.blob, variant, width, b, p)  # letters over the WHOLE dictionary
        self.setup_s = time.perf_counter() - t0
        self.n_all = n_all
        self.lo, self.hi = shard_bounds(n_all, parts, part)
        self.sblob, self.soffs = shard_of(self.blob, self.offs, self.lo, self.hi) if parts > 1 else (self.blob, self.offs)
        self.nq = len(self.qoffs) - 1
        self.mean_len = float(self.offs[-1]) / max(n_all, 1)
        self.qmean_len = float(self.qoffs[-1]) / max(self.nq, 1)

    def cell_name(self) -> str:
        from paper_1711_08475_b200.corpus import CELLS

        v, w, b, p, m = CELLS[self.cfg][self.cell]
        extra = f" b={b}" if v.name == "Count" else (f" p={p}" if v.name == "Position" else "")
        return f"{v.name}-{w}{extra} {m.name} k=1"

    def config(self, n_gpus: int) -> dict:
        """The `config` object of both arms' JSON lines (identical keys)."""
        return {"workload": f"config{self.cfg}", "cell": self.cell_name(), "n_words": self.n_all,
                "n_queries": self.nq, "mean_word_len": round(self.mean_len, 3),
                "mean_query_len": round(self.qmean_len, 3), "k": 1, "length_prefilter": True,
                "query_stats": True, "letters": self.scheme.letters().symbols().decode("latin-1"),
                "l2": L2_NOTE, "parallelism": f"dict-shard x{n_gpus}",
                "scaling_mode": "strong" if self.strong else "weak"}


_PINNED = []  # owners of pinned host storage


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """Copy of `a` in page-locked host memory (torch pinned allocator)."""
    import torch

    t = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    _PINNED.append(t)
    v = t.numpy()[: a.nbytes].view(a.dtype)
    v[:] = a
    return v


def reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def cpu_reference_rate(w: Workload, budget_s: float, threads: int):
    """Reference CPU scan (oracle/_ref, else the C restatement) of the whole
    dictionary on a bounded, evenly spaced query sample; returns (pairs/s,
    kind, sample description).  Letters and scheme are the GPU arm's."""
    from oracle.oracle import Oracle, Reference, oscheme
    from paper_1711_08475_b200.corpus import subsample

    blob, offs, qblob, qoffs, scheme, metric = w.blob, w.offs, w.qblob, w.qoffs, w.scheme, w.metric
    n, nq = len(offs) - 1, len(qoffs) - 1
    if Reference.available():
        ref = Reference()
        t0 = time.perf_counter()
        d = ref.dictionary(blob, offs, int(scheme.variant()), scheme.letters().symbols(),
                           scheme.bits_per_count() or 2, scheme.bits_per_position() or 3)
        build_s = time.perf_counter() - t0
        kind = "reference"
        run = lambda qb, qo: d.query_batch(qb, qo, int(metric), 1, True, True, threads)  # noqa: E731
    else:
        orc = Oracle()
        osch = oscheme(int(scheme.variant()), scheme.letters().symbols(), scheme.width(),
                       scheme.bits_per_count() or 2, scheme.bits_per_position() or 3)
        kind, build_s = "port", 0.0
        run = lambda qb, qo: orc.query_batch(blob, offs, qb, qo, osch, int(metric), 1, True, True, threads)  # noqa: E731

    def rate(budget):
        # calibrate on a small sample, then size the timed sample to the budget
        step = max(1, nq // (2 * threads))
        qb, qo, idx = subsample(qblob, qoffs, step)
        t0 = time.perf_counter()
        run(qb, qo)
        per_query = (time.perf_counter() - t0) / max(len(idx), 1)
        want = int(min(nq, max(threads, budget / max(per_query, 1e-9))))
        step = max(1, nq // want)
        qb, qo, idx = subsample(qblob, qoffs, step)
        t0 = time.perf_counter()
        run(qb, qo)
        dt = time.perf_counter() - t0
        sample = (f"every {step}th query ({len(idx)} of {nq}) x all {n} words, one pass, {dt:.1f} s "
                  f"(reference dictionary construction {build_s:.1f} s, untimed)")
        return len(idx) * n / dt, sample

    return rate, kind


def reference_arm(args) -> None:
    """The reference's CPU scan on all host threads, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1711_08475_b200 import _lib

    w = Workload(args.config, args.cell)
    threads = _lib.host_threads()
    rate, kind = cpu_reference_rate(w, 0, threads)
    rates, sample = [], ""
    per_step = max(2.0, 60.0 / max(args.steps, 1))
    for i in range(args.warmup + args.steps):
        r, sample = rate(per_step if i >= args.warmup else 1.0)
        if i >= args.warmup:
            rates.append(r)
    assert _lib._fpg is None, "the reference arm must not load libfpg.so"
    value = statistics.mean(rates)
    line = {"metric": METRIC, "value": value, "unit": "comparisons/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * w.nq * w.n_all / value,  # one full batch at the sampled rate
            "higher_is_better": True, "scaling": "strong" if w.strong else "weak", "vs_baseline": None,
            "dtype": "u8", "data": f"synthetic (seeded generator, config {args.config}; see corpus.py)",
            "config": w.config(args.gpus),
            "cpu_baseline": {"value": value, "unit": "comparisons/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": "comparisons/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "libfpg_loaded": False}
    print(json.dumps(line), flush=True)


def bench_devices(n: int) -> tuple[int, ...]:
    """Devices of the one-process N-GPU run: FPG_BENCH_DEVICES ("0,0") or
    0..n-1; fails loudly when fewer than n GPUs are present."""
    import torch

    env = os.environ.get("FPG_BENCH_DEVICES")
    if env:
        devs = tuple(int(x) for x in env.split(","))
        if len(devs) != n:
            raise SystemExit(f"FPG_BENCH_DEVICES lists {len(devs)} devices, --gpus is {n}")
        return devs
    have = torch.cuda.device_count()
    if have < n:
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible "
                         "(set FPG_BENCH_DEVICES to place several shards on one device)")
    return tuple(range(n))


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    world, rank, local = dist_env()
    import torch

    if world > 1:
        import torch.distributed as dist

        if world != args.gpus:
            raise SystemExit(f"torchrun WORLD_SIZE={world} but --gpus {args.gpus}")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        devices = (local,)
    else:
        devices = bench_devices(args.gpus)
    n_gpus = args.gpus

    from paper_1711_08475_b200 import GpuFingerprintedDictionary, QueryOptions
    from paper_1711_08475_b200._lib import host_threads

    w = Workload(args.config, args.cell, parts=world, part=rank)
    opt = QueryOptions(w.metric, 1, True, True)
    dev0 = devices[0]
    torch.cuda.set_device(dev0)
    d = GpuFingerprintedDictionary((w.sblob, w.soffs), w.scheme, devices=devices, id_base=w.lo, keep_words=False)
    build_s = d.build_seconds()
    nsh = len(devices)
    batch = d.batch()
    batch.upload(w.qblob, w.qoffs)
    flush = None
    if not args.no_flush:
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev0}")

    plan_ms = None

    def barrier():
        for dv in set(devices):
            torch.cuda.synchronize(dv)
        if world > 1:
            torch.distributed.barrier()

    for i in range(args.warmup):
        batch.run(opt, want_stats=True)
        if i == 0:  # the first run built the tile plan; the later ones reuse it
            plan_ms = max(batch.timing(s).get("plan_ms", 0.0) for s in range(nsh))
    clocks = Clocks(dev0)
    clocks.start()
    step_ms, shard_ms, filt_ms, ver_ms, launches = [], [], [], [], 0

    barrier()
    clocks.open()
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the event-timed run
            torch.cuda.synchronize(dev0)
        batch.run(opt, want_stats=True)
        ts = [batch.timing(s) for s in range(nsh)]
        step_ms.append(max(t["run_ms"] for t in ts))  # shards run concurrently: the slowest one
        shard_ms.append([t["run_ms"] for t in ts])
        filt_ms.append([t["filter_ms"] for t in ts])
        ver_ms.append([t.get("verify_ms", 0.0) for t in ts])
        launches += sum(t["launches"] for t in ts)
    barrier()
    clocks.close()
    clk = clocks.stop()
    t_last = [batch.timing(s) for s in range(nsh)]
    csr, st = batch.download()
    total_ms = reduce_max(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    logical_pairs_all = float(w.nq) * w.n_all  # Q x N of the whole (sharded or replicated) job
    value = logical_pairs_all * args.steps / (total_ms / 1e3)

    # e2e through the public API with pinned host buffers
    qb_p, qo_p = pinned_copy(w.qblob), pinned_copy(w.qoffs)
    e2e = None
    if not args.no_e2e:
        gather, phases = [], []
        if world == 1:
            def e2e_step():
                t0 = time.perf_counter()
                batch.upload(qb_p, qo_p)  # H2D
                t1 = time.perf_counter()
                batch.run(opt, want_stats=True)
                t2 = time.perf_counter()
                out = batch.download()  # D2H + host gather of the shard rows + QueryStats
                t3 = time.perf_counter()
                gather.append(batch.host_ms()["assemble_ms"])
                phases.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
                return out[0]
        else:
            cap = int(csr.offsets[-1]) if csr.offsets is not None else 0
            h_out = (torch.empty(w.nq + 1, dtype=torch.int64, pin_memory=True),
                     torch.empty(max(int(reduce_sum(cap, world)) * 2, 1), dtype=torch.int32, pin_memory=True))

            def e2e_step():
                batch.upload(qb_p, qo_p)  # H2D
                batch.run(opt, want_stats=True)
                t1 = time.perf_counter()
                out = _gather_merge(batch, h_out)  # NCCL gather, device merge, D2H on rank 0
                gather.append((time.perf_counter() - t1) * 1e3)
                return out
        # warm up exactly like the timed loop: the previous step's result stays
        # alive while the next one is produced, so two sets of pinned result
        # blocks rotate (a fresh 340 MB page-locked allocation costs ~170 ms)
        last = None
        for _ in range(max(2, args.warmup)):
            last = e2e_step()
        barrier()
        e2e_s = 0.0
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
                torch.cuda.synchronize(dev0)
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            last = e2e_step()
            e2e_s += time.perf_counter() - t0
        barrier()
        e2e_s = reduce_max(e2e_s, world)
        if rank == 0 and world == 1:
            assert np.array_equal(last.word_ids, csr.word_ids), "e2e and staged results differ"
        h2d = int(w.qblob.nbytes + w.qoffs.nbytes)
        n_match = int(last[1].size) if world > 1 and last is not None else int(csr.offsets[-1])
        d2h = int(8 * (w.nq + 1) + 4 * n_match + (8 * 5 * w.nq if world == 1 else 0))
        e2e = {"value": logical_pairs_all * args.steps / e2e_s, "unit": "comparisons/s",
               "h2d_bytes_per_step": h2d * (world if world > 1 else 1), "d2h_bytes_per_step": d2h,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "gather_ms_per_step": statistics.mean(gather[-args.steps:]) if gather else None,
               "phases_ms": ({k: statistics.mean(p[i] for p in phases[-args.steps:])
                              for i, k in enumerate(("upload", "run", "download"))} if phases else None),
               "download_ms_steps": [round(p[2], 2) for p in phases[-args.steps:]] if phases else None,
               "gather": ("host: libfpg.so concatenates the shard rows (fpg_batch_download)" if world == 1 else
                          "device: NCCL p2p of the ranks' CSRs to rank 0 + fpg_csr_merge_device, one D2H"),
               "l2": L2_NOTE}

    # the reference's per-pattern call (query_into, dictionary.hpp:75-118)
    # through the same C ABI: one batch round trip per pattern
    single_ms = None
    if world == 1 and not args.no_e2e:
        pats = [bytes(w.qblob[int(w.qoffs[i]):int(w.qoffs[i + 1])]) for i in range(0, min(w.nq, 64), 4)]
        d.query(pats[0], opt)
        t0 = time.perf_counter()
        for pat in pats:
            d.query(pat, opt)
        single_ms = 1e3 * (time.perf_counter() - t0) / len(pats)

    if rank != 0:
        return
    sms = torch.cuda.get_device_properties(dev0).multi_processor_count
    sm_mhz = clk.get("sm_max_mhz") or 1965.0
    # roofline of the dominant kernel (K2) on shard 0: the pairs it evaluated
    # per launch (length-compatible pairs minus those the weight window
    # skipped) / the launch's CUDA-event time, against
    # the ALU-pipe bound of the bit-sliced test
    t0s = t_last[0]
    filt_avg_ms = statistics.mean(f[0] for f in filt_ms)
    achieved = t0s["scanned_pairs"] / (filt_avg_ms / 1e3) / 1e12
    shape = d.scan_shape()
    # LOP3 per comparison, weighted over the sig' launch and the exact path's
    pairs_x = t0s.get("scanned_pairs_exact", 0)
    pairs_m = t0s["scanned_pairs"] - pairs_x
    ops = ((pairs_m * ops_per_comparison(w.scheme, shape["sig_fields"]) +
            pairs_x * ops_per_comparison(w.scheme, shape["sig_fields"], exact=True)) /
           max(pairs_m + pairs_x, 1))
    lop3_clk, lop3_basis = alu_peak()
    imad_clk = imad_peak()
    imads = ((pairs_m * imads_per_comparison(w.scheme, shape["sig_fields"]) +
              pairs_x * imads_per_comparison(w.scheme, shape["sig_fields"], exact=True)) / max(pairs_m + pairs_x, 1))
    popc_peak = sms * sm_mhz * 1e6 * POPC_PER_CLK_PER_SM / math.ceil(w.scheme.width() / 32) / 1e12
    if shape["sliced"]:
        # the pipe that binds: the ALU pipe (LOP3: the counters) or the FMA pipe
        # (IMAD: the query XOR of every plane); the position-code path has more
        # IMAD (30 per 32 pairs) than LOP3 (24)
        peak_alu = sms * sm_mhz * 1e6 * lop3_clk / ops / 1e12
        peak_fma = sms * sm_mhz * 1e6 * imad_clk / max(imads, 1e-9) / 1e12
        peak = min(peak_alu, peak_fma)
        bound = "int-alu" if peak_alu <= peak_fma else "int-fma"
        basis = (f"{sms} SMs x {sm_mhz:.0f} MHz x min({lop3_clk:.1f} LOP3/clk/SM / {ops:.3f} LOP3 per comparison, "
                 f"{imad_clk:.1f} IMAD/clk/SM / {imads:.3f} IMAD per comparison) ({lop3_basis}; bit-sliced test, "
                 f"{shape['sig_fields']} sig' planes; position-code-path pairs weighted with their own counts)")
    else:
        peak = popc_peak
        bound, basis = "int-xu", f"{sms} SMs x {sm_mhz:.0f} MHz x {POPC_PER_CLK_PER_SM} POPC/clk/SM / ceil(W/32)"
    traffic = profiled_traffic(f"config{args.config}", w.cell_name())
    # K3 (out-of-line byte verification, shard 0): HBM-bound.  Algorithmic
    # bytes per launch = the 16-byte candidate records read + one padded word
    # (its length bucket's stride) per candidate pair + an 8-byte key per match
    ver_avg_ms = statistics.mean(v[0] for v in ver_ms)
    hbm, hbm_basis = hbm_peak()
    w_stride = 16 * max(1, math.ceil(w.mean_len / 16))
    n_match0 = int(csr.offsets[-1]) if world == 1 and nsh == 1 else None
    ver_bytes = (16.0 * t0s.get("candidate_records", 0) * t0s.get("verify_rounds", 1) + float(w_stride) * t0s["candidates"] +
                 8.0 * (n_match0 or 0))
    verify = None
    if shape["sliced"] and ver_avg_ms > 0:
        gbs = ver_bytes / (ver_avg_ms * 1e6)
        verify = {"kernel": "k_verify (K3)", "bound": "hbm", "ms_per_step": ver_avg_ms, "algorithmic_bytes": ver_bytes,
                  "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "peak_basis": hbm_basis,
                  "traffic": profiled_traffic(f"config{args.config}", w.cell_name() + " k_verify"),
                  "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
                  "note": "the warps claim the records in stream order, so the candidate words hit L2 and the "
                          "DRAM traffic is essentially the records; ncu shows the kernel issue-bound (DESIGN.md section 3)",
                  "candidate_records": t0s.get("candidate_records", 0), "rounds": t0s.get("verify_rounds", 1),
                  "bytes_basis": f"16 B per record (upper bound: records of the largest round x rounds) + {w_stride} B "
                                 "per candidate word (random 32-byte sectors in practice) + 8 B per match key"}
    line = {
        "metric": METRIC, "value": value, "unit": "comparisons/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if w.strong else "weak", "vs_baseline": None,
        "dtype": "u8", "data": f"synthetic (seeded generator, config {args.config}; see corpus.py)",
        "config": w.config(n_gpus),
        "queries_per_s": w.nq * args.steps / (total_ms / 1e3),
        "executed_pairs_per_step": sum(t["executed_pairs"] for t in t_last),
        "evaluated_pairs_per_step": sum(t["scanned_pairs"] for t in t_last),
        "exact_path_pairs_per_step": sum(t.get("scanned_pairs_exact", 0) for t in t_last),
        "survivors_per_step": sum(t["survivors"] for t in t_last),
        "verifier_candidates_per_step": sum(t["candidates"] for t in t_last),
        "matches_per_step": int(csr.offsets[-1]) if world == 1 else None,
        "shard_ms_per_step": [statistics.mean(s[i] for s in shard_ms) for i in range(nsh)],
        "host_plan_ms": plan_ms, "single_query_ms": single_ms,
        "construction_s": build_s, "setup_s": w.setup_s,
        "construction": construction_roofline(d),
        "gpu_launches": launches,
        "e2e": e2e,
        "verify": verify,
        "roofline": {"bound": bound, "kernel": "k_slice (K2 filter)" if shape["sliced"] else "k_scan (K2)",
                     "achieved": achieved, "peak": peak, "unit": "Tcmp/s", "frac": achieved / peak,
                     "pairs_basis": "pairs K2 evaluated (length-compatible minus weight-window skips)",
                     "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
                     "peak_basis": basis,
                     "peak_alu": peak_alu if shape["sliced"] else None, "peak_fma": peak_fma if shape["sliced"] else None,
                     "popc_equiv_peak": popc_peak, "popc_equiv_frac": achieved / popc_peak,
                     "filter_ms_per_launch": filt_avg_ms, "filter_share_of_step": filt_avg_ms / ms_per_step},
        "clocks": clk,
    }
    if not args.no_cpu_baseline and n_gpus == 1:
        rate, kind = cpu_reference_rate(w, args.cpu_seconds, host_threads())
        r, sample = rate(args.cpu_seconds)
        line["cpu_baseline"] = {"value": r, "unit": "comparisons/s", "cores": host_threads(), "kind": kind,
                                "sample": sample}
    print(json.dumps(line), flush=True)


def _gather_merge(batch, h_out):
    """One process per GPU: this rank's device CSR to rank 0 over NCCL, merged
    there on the GPU and copied to the host (sharding.query_batch_distributed
    without the run, which the caller already timed)."""
    import torch
    import torch.distributed as dist

    from paper_1711_08475_b200.sharding import device_tensors, gather_rows, merge_device

    csr = batch.device_csr(0)
    off, ids = device_tensors(csr)
    parts = gather_rows(off, ids, dst=0)
    if dist.get_rank() != 0:
        return None
    m_off, m_ids = merge_device(parts, csr["nq"], csr["device"])
    h_off, h_ids = h_out[0][: m_off.numel()], h_out[1][: m_ids.numel()]
    h_off.copy_(m_off, non_blocking=True)
    h_ids.copy_(m_ids, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h_off.numpy().view(np.uint64), h_ids.numpy().view(np.uint32)


if __name__ == "__main__":
    main()
