#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a launch list (--metrics
gpu__time_duration.sum --csv) and/or a --set full report of one kernel.

usage: tools/ncu_summary.py launches <launches.csv>
       tools/ncu_summary.py report <prof.ncu-rep> [<src-lines>]
       tools/ncu_summary.py traffic <prof.ncu-rep> "<workload> <cell>" profiles/traffic.json
       tools/ncu_summary.py sass <prof.ncu-rep>   (executed SASS by opcode and hottest blocks)
"""
import collections
import csv
import io
import subprocess
import sys

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                unit = d.get("Metric Unit", "ns")
                v = float(d["Metric Value"].replace(",", ""))
                v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
                k = d["Kernel Name"].split("(")[0][:90]
                agg[k][0] += 1
                agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total us':>10} {'avg us':>9} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:9.1f} {100 * v[1] / tot:5.1f}%  {k}")
    print(f"total device time of listed launches: {tot:.1f} us (serialised, cold-cache; compare shares)")


def report(path, nlines=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "?"))
    for k in RAW_KEYS:
        if k in d:
            print(f"  {k} = {d[k]} {u.get(k, '')}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    if st:
        print("  stall reasons (warps per issue-active cycle): " +
              ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    out, fname = [], None
    for r in csv.reader(io.StringIO(src)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] and r[0].isdigit() and len(r) > 7:
            def num(x):
                try:
                    return int(x)
                except ValueError:
                    return 0
            out.append((num(r[7]), num(r[4]), fname, int(r[0]), r[1].strip()[:80]))
    ti = sum(o[0] for o in out) or 1
    ts = sum(o[1] for o in out) or 1
    print(f"  warp instructions executed: {ti}; stall samples: {ts}")
    print("  top source lines by stall samples (instr share / sample share):")
    for o in sorted(out, key=lambda x: -x[1])[:nlines]:
        print(f"    {100 * o[0] / ti:5.1f}% {100 * o[1] / ts:5.1f}%  {o[2]}:{o[3]}  {o[4]}")


def traffic(path, key, out_json):
    """Record dram__bytes_read.sum + dram__bytes_write.sum of the captured
    launch under `key` ("<workload> <cell>") in out_json (bench.py reads it)."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = sum(float(d[k].replace(",", "")) * scale.get(u[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    db = json.load(open(out_json)) if os.path.exists(out_json) else {}
    db[key] = {"kernel": d.get("Kernel Name", "?"), "dram_bytes": tot, "report": os.path.basename(path),
               "duration_us": float(d["gpu__time_duration.sum"].replace(",", "")) *
               {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(
                   u["gpu__time_duration.sum"], 1.0)}
    json.dump(db, open(out_json, "w"), indent=1, sort_keys=True)
    print(key, db[key])


def sass(path, nblocks=12):
    """Executed warp instructions by SASS opcode, and the hottest straight-line
    blocks (runs of instructions with equal execution counts) with their mix."""
    import re
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = next(r for r in rows if "Instructions Executed" in r)
    data = rows[rows.index(hdr) + 1:]
    ie, sc = hdr.index("Instructions Executed"), hdr.index("Source")

    def op(txt):
        t = re.sub(r"^@!?U?P\w+\s+", "", txt.strip())
        return t.split()[0] if t else "?"
    tot, byop, blocks, cur = 0, collections.Counter(), [], None
    for i, r in enumerate(data):
        if len(r) <= max(ie, sc):
            continue
        n = int(r[ie] or 0)
        tot += n
        byop[op(r[sc])] += n
        if cur and cur[0] == n:
            cur[2].append(op(r[sc]))
        else:
            cur = [n, i, [op(r[sc])]]
            blocks.append(cur)
    print(f"warp instructions executed: {tot}")
    for o, n in byop.most_common(25):
        print(f"  {o:22s} {n:14d} {100 * n / max(tot, 1):5.1f}%")
    print("hottest blocks (start index, executions, length, share, mix):")
    for n, i, ops in sorted(blocks, key=lambda b: -b[0] * len(b[2]))[:nblocks]:
        mix = ", ".join(f"{k} {v}" for k, v in collections.Counter(ops).most_common(6))
        print(f"  @{i:5d} x{n:10d} len {len(ops):4d} {100 * n * len(ops) / max(tot, 1):5.1f}%  {mix}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "sass":
        sass(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        report(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
