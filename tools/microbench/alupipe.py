#!/usr/bin/env python
"""Builds and runs tools/microbench/alupipe.cu on the GPU, samples the SM
clock with NVML while it runs, and writes profiles/alu_peak.json (bench.py's
ALU-pipe roofline denominator) plus the raw output to profiles/<tag>_alupipe.txt.

usage: python tools/microbench/alupipe.py <tag>"""
import json
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
HERE = Path(__file__).resolve().parent


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    exe = HERE / "alupipe"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                    str(HERE / "alupipe.cu")], check=True)
    sass = subprocess.run(["cuobjdump", "-sass", str(exe)], capture_output=True, text=True).stdout
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk, stop = [], [False]

    def sample():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.005)
    t = threading.Thread(target=sample, daemon=True)
    t.start()
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    stop[0] = True
    t.join()
    mhz = statistics.median(clk) if clk else float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
    sms = 148
    res = {}
    for line in out.splitlines():
        if "thread-ops/s=" in line and not line.startswith("--"):
            name = line.split()[0]
            ops = float(line.split("thread-ops/s=")[1].split()[0])
            res.setdefault(name, ops)  # the first (full-occupancy) run of each kernel
        if line.startswith("device"):
            sms = int(line.split("SMs=")[1].split()[0])
    per_clk = {k: v / (sms * mhz * 1e6) for k, v in res.items()}
    text = out + f"\nSM clock during the run (NVML median of {len(clk)} samples): {mhz:.0f} MHz\n"
    text += "".join(f"{k}: {v:.2f} thread-ops/clk/SM\n" for k, v in per_clk.items())
    text += "SASS opcode counts of the binary: " + ", ".join(
        f"{op} {sass.count(op + ' ')}" for op in ("LOP3.LUT", "IMAD", "LDS")) + "\n"
    (ROOT / "profiles" / f"{tag}_alupipe.txt").write_text(text)
    print(text)
    rec = {"lop3_per_clk_per_sm": round(per_clk["LOP3"], 2), "imad_per_clk_per_sm": round(per_clk["IMAD"], 2),
           "lop3_imad_dual_per_clk_per_sm": round(per_clk["LOP3+IMAD"], 2),
           "basis": f"measured on B200 ({tag}, tools/microbench/alupipe.cu, 16 chains x 64 warps/SM, "
                    f"{mhz:.0f} MHz): profiles/{tag}_alupipe.txt",
           "sm_mhz": mhz}
    (ROOT / "profiles" / "alu_peak.json").write_text(json.dumps(rec, indent=1) + "\n")


if __name__ == "__main__":
    main()
