#!/usr/bin/env python
"""Benchmark of the k=1 fingerprint-filtered query x dictionary scan.

Metric (BASELINE.json:2): logical query x word comparisons per second,
Q * N per batch (the reference's pair denominator, bench.hpp:157-161),
whole job over all GPUs.  Default workload = config 2 (BASELINE.json:8,
configs[1]): 1e6 uniform a-z words, L~U[4,20], 10,000 queries, count-16
fingerprints (b=2, 8 common letters), Levenshtein, k=1, length prefilter on,
per-query QueryStats on.  One step = one batch through the scan.

Multi-GPU (torchrun, one process per GPU): weak scaling.  Rank r owns
dictionary shard r = words [r*N, (r+1)*N) of config 2's seeded stream (shard
0 IS config 2's dictionary); every rank scans the same 10,000 queries;
word ids are rebased by r*N; results land in each rank's host memory.
No data-path collective.  Times are CUDA-event device times, max over ranks.

  value  device-resident: inputs already in HBM (fpg_batch_run only)
  e2e    through the public C ABI call fpg_query_batch with pinned host
         buffers: H2D of the queries, scan, D2H of the CSR + stats

--impl reference runs the reference's own CPU implementation
(oracle/_ref/libfpref.so: /root/reference headers, FingerprintedDictionary::
query_into) on all host threads over a bounded query sample of the same
workload, on rank 0 only.
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

POPC_PER_CLK_PER_SM = 16  # measured: tools/microbench/intpipe.cu (profiles/r01_phase0.txt)
ALU_PER_CLK_PER_SM = 64   # LOP3 issue: 16 lanes/clk/SMSP (B300_MICROARCH.md "Pipe rates")


def ops_per_comparison(scheme, sig_fields: int) -> float:
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
    return (ors + csa(nf + extra) + csa(sig_fields) + 1) / 32.0


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
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cell", type=int, default=0, help="index into corpus.CELLS[config]")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
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


def workload(cfg: int, cell: int, rank: int, world: int):
    from paper_1711_08475_b200.corpus import CELLS, CONFIGS, generate_dictionary, generate_queries, make_scheme

    c = CONFIGS[cfg]
    n = c.n_words // world if cfg == 5 else c.n_words  # cfg5: strong (the 64M dict split); else weak
    first = rank * n
    base_blob, base_offs = generate_dictionary(cfg, n=n if cfg != 5 else min(n, 8_000_000), first=0)
    blob, offs = (base_blob, base_offs) if first == 0 and cfg != 5 else generate_dictionary(cfg, n=n, first=first)
    qblob, qoffs = generate_queries(cfg, base_blob, base_offs, nq=c.n_queries)
    variant, width, b, p, metric = CELLS[cfg][cell]
    scheme = make_scheme(base_blob, variant, width, b, p)  # letters from the base (config) dictionary
    return c, blob, offs, qblob, qoffs, scheme, metric, first, n


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


def cpu_reference_rate(blob, offs, qblob, qoffs, scheme, metric, budget_s: float, threads: int):
    """Reference CPU scan (oracle/_ref, else the C restatement) on a bounded
    query sample; returns (pairs/s, kind, sample description, threads)."""
    from oracle.oracle import Oracle, Reference, oscheme
    from paper_1711_08475_b200.corpus import subsample

    n = len(offs) - 1
    nq = len(qoffs) - 1
    if Reference.available():
        ref = Reference()
        d = ref.dictionary(blob, offs, int(scheme.variant()), scheme.letters().symbols(),
                           scheme.bits_per_count() or 2, scheme.bits_per_position() or 3)
        kind = "reference"
        run = lambda qb, qo: d.query_batch(qb, qo, int(metric), 1, True, True, threads)  # noqa: E731
    else:
        orc = Oracle()
        osch = oscheme(int(scheme.variant()), scheme.letters().symbols(), scheme.width(),
                       scheme.bits_per_count() or 2, scheme.bits_per_position() or 3)
        kind = "port"
        run = lambda qb, qo: orc.query_batch(blob, offs, qb, qo, osch, int(metric), 1, True, True, threads)  # noqa: E731
    # calibrate on a small sample, then size the timed sample to the budget
    step = max(1, nq // (4 * threads))
    qb, qo, idx = subsample(qblob, qoffs, step)
    t0 = time.perf_counter()
    run(qb, qo)
    dt = time.perf_counter() - t0
    per_query = dt / max(len(idx), 1)
    want = int(min(nq, max(threads, budget_s / max(per_query, 1e-9))))
    step = max(1, nq // want)
    qb, qo, idx = subsample(qblob, qoffs, step)
    t0 = time.perf_counter()
    run(qb, qo)
    dt = time.perf_counter() - t0
    pairs = len(idx) * n
    sample = f"every {step}th query ({len(idx)} of {nq}) x all {n} words, one pass, {dt:.1f} s"
    return pairs / dt, kind, sample, dt


def main():
    args = parse()
    world, rank, local = dist_env()
    from paper_1711_08475_b200._lib import host_threads

    if args.impl == "reference":
        if rank != 0:
            return
        c, blob, offs, qblob, qoffs, scheme, metric, first, n = workload(args.config, args.cell, 0, 1)
        threads = host_threads()
        rates = []
        sample = kind = ""
        for i in range(args.warmup + args.steps):
            budget = max(2.0, 60.0 / (args.warmup + args.steps)) if i >= args.warmup else 1.0
            r, kind, sample, _ = cpu_reference_rate(blob, offs, qblob, qoffs, scheme, metric, budget, threads)
            if i >= args.warmup:
                rates.append(r)
        value = statistics.mean(rates)
        line = {"metric": "k=1 query x word comparisons/s (logical Q*N)", "value": value, "unit": "comparisons/s",
                "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * c.n_queries * n / value,  # one full batch at the sampled rate "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u8", "data": "synthetic (seeded generator, config %d)" % args.config,
                "config": {"workload": f"config{args.config}", "cell": _cell_name(args.config, args.cell),
                           "n_words": n, "n_queries": c.n_queries},
                "cpu_baseline": {"value": value, "unit": "comparisons/s", "cores": threads, "kind": kind,
                                 "sample": sample},
                "e2e": {"value": value, "unit": "comparisons/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local if world > 1 else 0

    from paper_1711_08475_b200 import GpuFingerprintedDictionary, QueryOptions

    c, blob, offs, qblob, qoffs, scheme, metric, first, n = workload(args.config, args.cell, rank, world)
    nq = len(qoffs) - 1
    opt = QueryOptions(metric, 1, True, True)
    d = GpuFingerprintedDictionary((blob, offs), scheme, devices=(dev,), id_base=first, keep_words=False)
    build_s = d.build_seconds()
    batch = d.batch()
    batch.upload(qblob, qoffs)
    flush = None
    if not args.no_flush:
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        batch.run(opt, want_stats=True)
    clocks = Clocks(dev)
    clocks.start()
    run_ms, filt_ms, launches, executed, survivors, candidates, scanned = [], [], 0, 0, 0, 0, 0
    barrier()
    clocks.open()
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the event-timed run
            torch.cuda.synchronize(dev)
        batch.run(opt, want_stats=True)
        t = batch.timing()
        run_ms.append(t["run_ms"])
        filt_ms.append(t["filter_ms"])
        launches += t["launches"]
        executed, survivors, candidates = t["executed_pairs"], t["survivors"], t["candidates"]
        scanned = t["scanned_pairs"]
    barrier()
    clocks.close()
    clk = clocks.stop()
    csr, st = batch.download()
    total_ms = reduce_max(sum(run_ms), world)
    ms_per_step = total_ms / args.steps
    logical_pairs_all = reduce_sum(float(nq) * n, world)  # Q x N over all shards
    value = logical_pairs_all * args.steps / (total_ms / 1e3)

    # e2e: public C ABI call with pinned host buffers (H2D + scan + D2H inside)
    qb_p, qo_p = pinned_copy(qblob), pinned_copy(qoffs)
    for _ in range(max(1, args.warmup)):
        d.query_batch((qb_p, qo_p), opt, per_query_stats=True)
    barrier()
    e2e_s, e2e_csr = 0.0, None
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
            torch.cuda.synchronize(dev)
        t0 = time.perf_counter()  # the call is blocking: H2D, scan, D2H, CSR assembly
        e2e_csr, _ = d.query_batch((qb_p, qo_p), opt, per_query_stats=True)
        e2e_s += time.perf_counter() - t0
    barrier()
    e2e_s = reduce_max(e2e_s, world)
    e2e_value = logical_pairs_all * args.steps / e2e_s

    assert np.array_equal(e2e_csr.word_ids, csr.word_ids), "e2e and staged results differ"
    h2d = int(qblob.nbytes + qoffs.nbytes)
    d2h = int(8 * (nq + 1) + 4 * int(csr.offsets[-1]) + 4 * nq)

    if rank != 0:
        return
    # roofline of the dominant kernel (K2): the pairs it evaluated per launch
    # (length-compatible pairs minus those skipped by the weight window) / the
    # launch's CUDA-event time, against the ALU-pipe bound of the bit-sliced
    # test
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = clk.get("sm_max_mhz") or 1965.0
    filt_avg_ms = statistics.mean(filt_ms)
    achieved = (scanned or executed) / (filt_avg_ms / 1e3) / 1e12
    shape = d.scan_shape()
    ops = ops_per_comparison(scheme, shape["sig_fields"])
    popc_peak = sms * sm_mhz * 1e6 * POPC_PER_CLK_PER_SM / math.ceil(scheme.width() / 32) / 1e12
    if shape["sliced"]:
        peak = sms * sm_mhz * 1e6 * ALU_PER_CLK_PER_SM / ops / 1e12
        bound, basis = "int-alu", (f"{sms} SMs x {sm_mhz:.0f} MHz x {ALU_PER_CLK_PER_SM} LOP3/clk/SM / "
                                   f"{ops:.3f} LOP3 per comparison (bit-sliced test, {shape['sig_fields']} sig' planes)")
    else:
        peak = popc_peak
        bound, basis = "int-xu", f"{sms} SMs x {sm_mhz:.0f} MHz x {POPC_PER_CLK_PER_SM} POPC/clk/SM / ceil(W/32)"
    traffic = profiled_traffic(f"config{args.config}", _cell_name(args.config, args.cell))
    line = {
        "metric": "k=1 query x word comparisons/s (logical Q*N)",
        "value": value, "unit": "comparisons/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": f"synthetic (seeded generator, config {args.config}; see corpus.py)",
        "config": {"workload": f"config{args.config}", "cell": _cell_name(args.config, args.cell),
                   "n_words_per_gpu": n, "n_queries": nq, "length_prefilter": True, "query_stats": True,
                   "l2": "flushed between steps (256 MB write)" if flush is not None else "not flushed",
                   "parallelism": f"dict-shard x{world}"},
        "queries_per_s": nq * args.steps / (total_ms / 1e3),
        "executed_pairs_per_step": executed, "evaluated_pairs_per_step": scanned, "survivors_per_step": survivors,
        "verifier_candidates_per_step": candidates,
        "matches_per_step": int(csr.offsets[-1]),
        "construction_s": build_s,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": "comparisons/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "l2": "flushed between steps"},
        "roofline": {"bound": bound, "kernel": "k_slice (K2 filter+verify)" if shape["sliced"] else "k_scan (K2)",
                     "achieved": achieved, "peak": peak, "unit": "Tcmp/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
                     "peak_basis": basis,
                     "popc_equiv_peak": popc_peak, "popc_equiv_frac": achieved / popc_peak,
                     "filter_ms_per_launch": filt_avg_ms, "filter_share_of_step": filt_avg_ms / ms_per_step},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        rate, kind, sample, dt = cpu_reference_rate(blob, offs, qblob, qoffs, scheme, metric,
                                                    args.cpu_seconds, host_threads())
        line["cpu_baseline"] = {"value": rate, "unit": "comparisons/s", "cores": host_threads(), "kind": kind,
                                "sample": sample}
    print(json.dumps(line), flush=True)


def _cell_name(cfg, cell):
    from paper_1711_08475_b200.corpus import CELLS

    v, w, b, p, m = CELLS[cfg][cell]
    extra = f" b={b}" if v.name == "Count" else (f" p={p}" if v.name == "Position" else "")
    return f"{v.name}-{w}{extra} {m.name} k=1"


if __name__ == "__main__":
    main()
